#!/bin/bash
# Round-end measurement bundle (run on the GPU box from the repo root):
# bench line, ncu launch list of the bench command, ncu --set full of the
# bench-config quantize / dequantize launches, summarised into gpurun_out/.
set -u
[ "${SKIP_BENCH:-0}" = 1 ] || timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
[ "${SKIP_LAUNCHES:-0}" = 1 ] || timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(quantize|dequant)_|k_attention' \
    --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
    > /dev/null 2>&1
# the bench-shape launches (time_codec compresses TC=2 chunks of 720 planes first)
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:'k_quantize_ring32' --launch-skip 4 -c 1 -o /tmp/codec_q python tools/time_codec.py > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:'k_dequant_ring32<.int.2, .int.2' --launch-skip 2 -c 1 -o /tmp/codec_d python tools/time_codec.py \
    > /dev/null 2>&1
python tools/ncu_summary.py /tmp/codec_q.ncu-rep /tmp/codec_d.ncu-rep > gpurun_out/ncu_full_codec.txt 2>&1
python tools/launch_list.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1
