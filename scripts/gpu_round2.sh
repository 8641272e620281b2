#!/bin/bash
# Round-2 measurement set: gpu tests, smoke, bench (config 2 + CPU baseline), reference arm,
# configs 3/4, ncu launch list, full captures of the top kernels, secondary sweep.
mkdir -p gpurun_out
T=${TAG:-r02c}
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pt_full.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for w in 3 4; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_w$w.json 2> gpurun_out/bench_w$w.err; echo "w$w rc=$?"
done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv $B > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches.csv > gpurun_out/${T}_launches.txt; head -14 gpurun_out/${T}_launches.txt
for k in kf32_train:prof_kf32 tc_train:prof_tc reduce_partials:prof_red adam_train:prof_adam; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${k%%:*} -s 2 -c 1 -o gpurun_out/${k##*:} $B > /dev/null 2>&1
  echo "ncu ${k} rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sample_prep -s 4 -c 2 -o gpurun_out/prof_prep $B > /dev/null 2>&1; echo "prep rc=$?"
timeout 1200 python scripts/bench_sweep.py > gpurun_out/${T}_sweep.json 2> gpurun_out/sweep.err; echo "sweep rc=$?"
