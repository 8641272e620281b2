#!/bin/bash
# Full ncu captures of the top kernels of the bench step + a config-4 bench line.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 python -m pytest tests -m gpu -q -x -k "sharded or config1" > gpurun_out/pt2.log 2>&1; tail -2 gpurun_out/pt2.log
for k in ${KERNELS:-kf32_train:prof_kf32 tc_train:prof_tc sample_prep:prof_prep}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${k%%:*} -s 2 -c 1 -o gpurun_out/${k##*:} $B > /dev/null 2>&1
  echo "ncu ${k} rc=$?"
done
if [ -n "$W4" ]; then
  timeout 900 python bench.py --workload 4 --steps 10 --warmup 3 --cpu-seconds 20 > gpurun_out/bench_w4.json 2> gpurun_out/bench_w4.err; echo "w4 rc=$?"
  head -c 1500 gpurun_out/bench_w4.json; tail -5 gpurun_out/bench_w4.err
fi
ls -la gpurun_out
