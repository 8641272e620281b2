#!/bin/bash
# Round profile capture (run under gpurun): launch list of the bench command
# and one full ncu capture of the fused kernel in the bench configuration.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt
ncu --set full --clock-control none --import-source on -k regex:mlp_kernel -s 2 -c 1 -o gpurun_out/prof_mlp \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sample_rays -s 2 -c 1 -o gpurun_out/prof_rays \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:adam_train -s 2 -c 1 -o gpurun_out/prof_adam \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
