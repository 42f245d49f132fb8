cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/probe_regress.py c2 > gpurun_out/probe_c2.log 2>&1
timeout 400 python tools/probe_regress.py c3 > gpurun_out/probe_c3.log 2>&1
timeout 300 python -m pytest tests/test_gpu_configs.py -x -q -m gpu -k "headline" > gpurun_out/t_head.log 2>&1
FGFRFT_STEP_SLICES=6 timeout 300 python -m pytest tests/test_gpu_configs.py -x -q -m gpu -k "headline" >> gpurun_out/t_head.log 2>&1
cat gpurun_out/probe_c2.log gpurun_out/probe_c3.log | cut -c1-400; tail -3 gpurun_out/t_head.log
