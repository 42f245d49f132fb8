mkdir -p gpurun_out/c5
ncu --set full --clock-control none --import-source on -k regex:"batch_dlda" -c 1 -o gpurun_out/c5/batch python tools/bench_configs.py --configs 5 > gpurun_out/c5/ncu.log 2>&1
