cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/t_batch.log 2>&1; echo "rc $?" >> gpurun_out/t_batch.log
tail -30 gpurun_out/t_batch.log
timeout 300 python tools/bench_configs.py --configs 5 > gpurun_out/c5.log 2>&1
FGFRFT_BATCH_FWD=2 FGFRFT_BATCH_DLDA=0 timeout 300 python tools/bench_configs.py --configs 5 >> gpurun_out/c5.log 2>&1
tail -c 1500 gpurun_out/c5.log
