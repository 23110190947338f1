timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_dequant_stream<.int.2, .int.2, .bool.1" --launch-skip 2 -c 1 -o /tmp/d python tools/time_codec.py > /tmp/d.log 2>&1
ncu -i /tmp/d.ncu-rep --page source --csv --print-source sass > gpurun_out/dsrc.csv 2>/dev/null
ncu -i /tmp/d.ncu-rep --page raw --csv > gpurun_out/draw.csv 2>/dev/null
ncu -i /tmp/d.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/dsrc_mixed.csv 2>/dev/null
tail -2 /tmp/d.log
