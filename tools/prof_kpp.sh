timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_kmeanspp" --launch-skip ${SKIP:-0} -c 1 -o /tmp/k python tools/prof_encode.py > /tmp/k.log 2>&1
ncu -i /tmp/k.ncu-rep --page source --csv --print-source sass > gpurun_out/ksrc.csv 2>/dev/null
ncu -i /tmp/k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ksrc_mixed.csv 2>/dev/null
ncu -i /tmp/k.ncu-rep --page raw --csv > gpurun_out/kraw.csv 2>/dev/null
