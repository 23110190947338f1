timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_assign_tc" --launch-skip ${SKIP:-0} -c 1 -o /tmp/t python tools/prof_encode.py > /tmp/t.log 2>&1
ncu -i /tmp/t.ncu-rep --page source --csv --print-source sass > gpurun_out/tsrc.csv 2>/dev/null
ncu -i /tmp/t.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/tsrc_mixed.csv 2>/dev/null
ncu -i /tmp/t.ncu-rep --page raw --csv > gpurun_out/traw.csv 2>/dev/null
