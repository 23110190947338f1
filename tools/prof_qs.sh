# ncu --set full of the bench-shape quantize launch (time_codec compresses 14
# chunks first; skip those launches), per-line SASS counts -> gpurun_out/
TAG=${1:-q}
KREGEX=${2:-k_quantize_stream}
timeout 300 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"$KREGEX" --launch-skip 4 -c 1 -o gpurun_out/$TAG python tools/time_codec.py > gpurun_out/$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_mixed.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/$TAG.ncu-rep > gpurun_out/$TAG.txt 2>&1
