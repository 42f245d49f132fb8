cd $GRAFT_REPO_ROOT
E=gpurun_out/nd2; mkdir -p $E
PROBE_TRACE=1 timeout 600 python tools/probe_regress.py c2 > $E/c2_on.jsonl 2>&1
FGFRFT_NODE_XSIDE=0 timeout 600 python tools/probe_regress.py c2 > $E/c2_off.jsonl 2>&1
cut -c1-700 $E/c2_on.jsonl | head -3; cut -c1-200 $E/c2_off.jsonl | head -3
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_configs.py tests/test_gpu_window.py -m gpu -q -x > $E/pytest.log 2>&1; tail -3 $E/pytest.log
