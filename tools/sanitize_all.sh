#!/bin/bash
# compute-sanitizer over the pipelined kernels (tools/sanitize_smoke.py);
# logs -> gpurun_out/sanitize_<tool>_<variant>.log
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool variant env...
    local tool=$1 var=$2; shift 2
    env "$@" timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_smoke.py \
        > gpurun_out/sanitize_${tool}_${var}.log 2>&1
    echo "$tool/$var rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|errors' gpurun_out/sanitize_${tool}_${var}.log | tail -1)"
}
TOOLS=${TOOLS:-"memcheck synccheck racecheck"}
for tool in $TOOLS; do
    if [ $tool = memcheck ]; then   # compress under memcheck only at the 4-plane size
        run $tool default SAN_ONLY=compress,codec_q,attention,container
    else
        run $tool default
    fi
done
