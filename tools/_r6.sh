cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/t_batch.log 2>&1; echo "rc $?" >> gpurun_out/t_batch.log
tail -3 gpurun_out/t_batch.log
timeout 300 python tools/bench_configs.py --configs 5 > gpurun_out/c5.log 2>&1
tail -c 1000 gpurun_out/c5.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:batch_fwd_tc -s 2 -c 1 -o gpurun_out/c5fwd2 python tools/bench_configs.py --configs 5 > gpurun_out/ncu_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:batch_dlda_tc -s 2 -c 1 -o gpurun_out/c5bwd2 python tools/bench_configs.py --configs 5 >> gpurun_out/ncu_c5.log 2>&1
