cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
timeout 600 python tools/c3_step.py --steps 10 --warmup 3 --sweep "FGFRFT_DSYNTH=0;FGFRFT_DSYNTH=1;FGFRFT_DSYNTH=1&FGFRFT_PIPE_SPLIT=0.3;FGFRFT_PIPE_SPLIT=0.25,0.5;FGFRFT_PIPE_SPLIT=" > gpurun_out/c3sweep.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
tail -3 gpurun_out/gputest.log; tail -c 600 gpurun_out/bench.log
