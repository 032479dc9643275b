#!/bin/bash
# Usage (on the GPU box via gpurun): bash profiles/run_profile.sh TAG [bench args]
# 1) the plain bench command, 2) the ncu launch list of the same command,
# 3) one --set full capture of the fused kernel (the product path: merge in
#    its tail) and, when the path has one, of the separate merge kernel.
# Each ncu pass runs only after the identical plain command exited 0.
TAG=${1:-prof}
shift
ARGS=${@:-"--steps 5 --warmup 3 --no-cpu-baseline --no-side"}
CMD="python bench.py $ARGS"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ol_tc -s 4 -c 1 -o gpurun_out/${TAG}_fused $CMD > gpurun_out/${TAG}_ncu_fused.log 2>&1
if grep -q merge_sentences gpurun_out/${TAG}_launches.csv; then
  ncu --set full --clock-control none --import-source on -k regex:merge_sentences -s 4 -c 1 -o gpurun_out/${TAG}_merge $CMD > gpurun_out/${TAG}_ncu_merge.log 2>&1
fi
echo "profile done"
