#!/bin/bash
# Round-2 re-entry check: all -m gpu tests, smoke, bench + reference arm, config 3/4 lines, launch list, sweep.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pt_full.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pt_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for w in 3 4; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err; echo "w$w rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt; head -20 gpurun_out/launches_summary.txt
timeout 1200 python scripts/bench_sweep.py > gpurun_out/sweep.json 2> gpurun_out/sweep.err; echo "sweep rc=$?"; tail -3 gpurun_out/sweep.err
