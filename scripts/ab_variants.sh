# A/B of library build variants (scripts/bin/<name>/libvmap_b200.so) vs the main build, 2 rounds
for r in 1 2; do
  for v in main ${VARIANTS}; do
    if [ "$v" = main ]; then L=""; else L="VM_LIB=scripts/bin/$v/libvmap_b200.so"; fi
    env $L timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_v.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/b_v.json').read().strip().splitlines()[-1])
print('$v', 'ms/step', round(d['ms_per_step'],4), 'KF', round(d['roofline_kernels'][0]['kernel_ms']*1e3,1), 'KT', round(d['roofline_kernels'][1]['kernel_ms']*1e3,1))"
  done
done
