#!/bin/bash
# Usage (on the GPU box via gpurun): bash profiles/run_profile.sh TAG
# plain bench run, then the ncu launch list and one --set full capture of the
# fused kernel (each only after the same command exited 0 without ncu).
TAG=${1:-prof}
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ol_tc_kernel -s 4 -c 1 -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "profile rc=$?"
