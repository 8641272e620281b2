for v in "" "VM_KT_FIRST=1" "VM_KT_FIRST=2" "VM_NO_FORK=1"; do
  env $v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_order.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_order.json').read().strip().splitlines()[-1])
print('$v', 'ms/step', round(d['ms_per_step'],4), 'mlp', round(d['mlp_phase']['ms'],4), 'red+adam', round(d['mlp_phase']['reduce_adam_ms'],4), [round(r['kernel_ms'],4) for r in d['roofline_kernels']])"
done
