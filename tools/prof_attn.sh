timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_attention_pp4" --launch-skip 3 -c 1 -o /tmp/a python tools/time_attn.py > /tmp/a.log 2>&1
ncu -i /tmp/a.ncu-rep --page source --csv --print-source sass > gpurun_out/asrc.csv 2>/dev/null
ncu -i /tmp/a.ncu-rep --page raw --csv > gpurun_out/araw.csv 2>/dev/null
ncu -i /tmp/a.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/asrc_mixed.csv 2>/dev/null
tail -2 /tmp/a.log
