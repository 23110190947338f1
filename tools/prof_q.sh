timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"v5w<.int.2, .int.2, .bool.1, .int.768" --launch-skip 2 -c 1 -o /tmp/q python tools/time_codec.py > /tmp/q.log 2>&1
ncu -i /tmp/q.ncu-rep --page source --csv --print-source sass > gpurun_out/qsrc.csv 2>/dev/null
ncu -i /tmp/q.ncu-rep --page raw --csv > gpurun_out/qraw.csv 2>/dev/null
tail -2 /tmp/q.log
ncu -i /tmp/q.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/qsrc_mixed.csv 2>/dev/null
