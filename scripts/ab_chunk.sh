# A/B of the FFMA object kernel's work-item size (blocks per CTA; K-independent either way)
for c in 4 6 8 12 16; do
  VM_KF_CHUNK=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_chunk.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_chunk.json').read().strip().splitlines()[-1])
print('chunk $c', 'ms/step', round(d['ms_per_step'],4), 'mlp', round(d['mlp_phase']['ms'],4), [round(r['kernel_ms'],4) for r in d['roofline_kernels']])"
  VM_NO_FORK=1 VM_KF_CHUNK=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_chunk.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_chunk.json').read().strip().splitlines()[-1])
print('  alone: KF', round(d['roofline_kernels'][0]['kernel_ms'],4))"
done
