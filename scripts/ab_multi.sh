# alternating A/B/C... of env settings given as arguments ("VAR=v VAR2=w"), $R rounds each
R=${R:-2}
for r in $(seq $R); do
  for v in "$@"; do
    env $v timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b_m.json 2>gpurun_out/b_m.err || tail -3 gpurun_out/b_m.err
    python -c "
import json; d=json.loads(open('gpurun_out/b_m.json').read().strip().splitlines()[-1])
print('[$v]', 'ms/step', round(d['ms_per_step'],4), 'mlp', round(d['mlp_phase']['ms'],4), [round(r['kernel_ms'],4) for r in d['roofline_kernels']])"
  done
done
