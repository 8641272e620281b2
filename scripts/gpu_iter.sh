#!/bin/bash
# One optimisation iteration: gpu tests, config-2 bench, ncu of the named kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pt_iter.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_iter.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_iter.json").read().strip().splitlines()[-1])
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]))
for r in d["roofline_kernels"]: print("  ", r["kernel"][:30], round(r["kernel_ms"]*1e3,1), "us frac", round(r["frac"],3))
print("  mlp", d["mlp_phase"])
PY
for k in ${KERNELS:-kf32_train:prof_kf32}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${k%%:*} -s 2 -c 1 -o gpurun_out/${k##*:} python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "ncu ${k} rc=$?"
done
