#!/bin/bash
# Round profile capture (run under gpurun; gpurun_out must stay < 64 MiB, so
# the per-kernel captures are split over two calls: `profile_round.sh 1|2`).
# Part 1: launch lists of the bench command (cold = ncu default cache flush,
# warm = --cache-control none) and full captures of KT and KF; part 2: the
# reduce, sampler and Adam kernels.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
if [ "${1:-1}" = "1" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv $B > /dev/null 2>&1
  python scripts/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 500 --csv \
      --log-file gpurun_out/launches_warm.csv $B > /dev/null 2>&1
  python scripts/launches.py gpurun_out/launches_warm.csv > gpurun_out/launches_warm_summary.txt
  K="tc_train:prof_tc mlp_kernel:prof_mlp"
else
  K="reduce_partials:prof_red sample_rays:prof_rays adam_train:prof_adam"
fi
for k in $K; do
  ncu --set full --clock-control none --import-source on -k regex:${k%%:*} -s 2 -c 1 -o gpurun_out/${k##*:} $B > /dev/null 2>&1
done
ls -la gpurun_out
