#!/bin/bash
# Full round check: all -m gpu tests, bench (config 2 with CPU baseline), the
# reference arm, config 3/4 bench lines, the secondary sweep.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pt_full.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pt_full.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for w in 3 4; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err; echo "w$w rc=$?"
done
timeout 1200 python scripts/bench_sweep.py > gpurun_out/sweep.json 2> gpurun_out/sweep.err; echo "sweep rc=$?"; tail -3 gpurun_out/sweep.err
