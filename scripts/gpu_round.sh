mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
for K in 50 200; do timeout 120 python scripts/kf_exp.py obj 30 $K; done > gpurun_out/kf.log 2>&1
timeout 120 python scripts/kf_exp.py both 30 >> gpurun_out/kf.log 2>&1
VM_KT_FIRST=1 timeout 120 python scripts/kf_exp.py both 30 >> gpurun_out/kf.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kf32 -s 3 -c 1 -o gpurun_out/prof_kf5 python scripts/kf_exp.py obj 3 > gpurun_out/ncu.log 2>&1
cat gpurun_out/kf.log
