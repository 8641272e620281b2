#!/bin/bash
# Full ncu captures (one launch each) of the step's top kernels, config 2, plus KF at config 4.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for k in ${KERNELS:-kf32_train:prof_kf32 tc_train:prof_tc reduce_partials:prof_red}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${k%%:*} -s 2 -c 1 -o gpurun_out/${k##*:} $B > /dev/null 2>&1
  echo "ncu ${k} rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sample_prep --launch-skip-before-match 0 -s 4 -c 2 -o gpurun_out/prof_prep $B > /dev/null 2>&1; echo "prep rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kf32_train -s 1 -c 1 -o gpurun_out/prof_kf32_w4 python bench.py --workload 4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "kf32 w4 rc=$?"
ls -la gpurun_out
