# A/B of the KF/KT schedule: persistent KF (work queue), KT-first with the weight image before the fork, chunk size
for v in "" "VM_KF_PERSIST=1" "VM_KT_FIRST=2" "VM_KF_PERSIST=1 VM_KT_FIRST=2" "VM_KF_PERSIST=1 VM_KT_FIRST=2 VM_KF_CHUNK=4" "VM_KF_PERSIST=1 VM_KF_CHUNK=4"; do
  env $v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_s.json 2>gpurun_out/b_s.err || tail -3 gpurun_out/b_s.err
  python -c "
import json; d=json.loads(open('gpurun_out/b_s.json').read().strip().splitlines()[-1])
print('$v', 'ms/step', round(d['ms_per_step'],4), 'mlp', round(d['mlp_phase']['ms'],4), [round(r['kernel_ms'],4) for r in d['roofline_kernels']])"
done
