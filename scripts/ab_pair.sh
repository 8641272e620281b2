# alternating A/B of two env settings ($A, $B), 3 rounds each
for r in 1 2 3; do
  for v in "$A" "$B"; do
    env $v timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b_p.json 2>gpurun_out/b_p.err || tail -3 gpurun_out/b_p.err
    python -c "
import json; d=json.loads(open('gpurun_out/b_p.json').read().strip().splitlines()[-1])
print('[$v]', 'ms/step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'mlp', round(d['mlp_phase']['ms'],4), [round(r['kernel_ms'],4) for r in d['roofline_kernels']])"
  done
done
