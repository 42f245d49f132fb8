cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/probe_regress.py c3 > gpurun_out/probe_c3.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
cat gpurun_out/probe_c3.log | cut -c1-400; tail -3 gpurun_out/gputest.log
