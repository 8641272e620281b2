#!/bin/bash
# -m gpu tests (selection via $SEL) + optional bench lines ($BENCH="2 3 4")
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x ${SEL:+-k "$SEL"} > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|error" gpurun_out/pt.log | tail -5
for w in $BENCH; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 ${CPU:---no-cpu-baseline} > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err; echo "bench w$w rc=$?"
  python -c "
import json;d=json.load(open('gpurun_out/bench_w$w.json'))
print('w$w', 'ms/step %.4f'%d['ms_per_step'], 'value %.0f'%d['value'], 'e2e %.0f'%d['e2e']['value'], [(k['kernel'][:12], round(k['kernel_ms'],4), round(k['frac'],3)) for k in d['roofline_kernels']], d['mlp_phase'])" 2>&1 | tail -2
done
