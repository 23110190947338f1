# ncu --set full of one bench-shape launch of kernel regex $2 (launch-skip $3)
# -> gpurun_out/$1.txt summary + per-instruction (cuda,sass) csv
TAG=$1; KREGEX=$2; SKIP=${3:-2}
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"$KREGEX" --launch-skip $SKIP -c 1 -o /tmp/$TAG python tools/time_codec.py > gpurun_out/$TAG.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_mixed.csv 2>/dev/null
python tools/ncu_summary.py /tmp/$TAG.ncu-rep > gpurun_out/$TAG.txt 2>&1
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
