#!/bin/bash
# One GPU round-trip: -m gpu tests, a bench line, the ncu launch list of the bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA -x > gpurun_out/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt.log
tail -3 gpurun_out/pt.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json | head -c 3000
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
cat gpurun_out/launches_summary.txt | head -30
