#!/bin/bash
# Final measurement set without full ncu captures (<64 MiB of outputs): tests, smoke, bench (config 2 +
# CPU baseline), reference arm, configs 3/4, ncu launch list, sweep, sanitizers.
mkdir -p gpurun_out
T=${TAG:-r02n}
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for w in 3 4; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_w$w.json 2> gpurun_out/bench_w$w.err; echo "w$w rc=$?"
done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
VM_BENCH_ALONE=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/${T}_launches.csv $B > /dev/null 2>&1
python scripts/launches.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.txt; head -14 gpurun_out/${T}_launches.txt
timeout 1200 python scripts/bench_sweep.py > gpurun_out/${T}_sweep.json 2> gpurun_out/sweep.err; echo "sweep rc=$?"
timeout 900 bash scripts/gpu_sanitize.sh > /dev/null 2>&1; cp gpurun_out/sanitizer.txt gpurun_out/${T}_sanitizer.txt; grep -E "SUMMARY" gpurun_out/${T}_sanitizer.txt
du -sh gpurun_out
