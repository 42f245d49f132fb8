# Iteration run: the fused-MSE tests, the packed / window / config suites, then the bench.
cd $GRAFT_REPO_ROOT
E=gpurun_out/it2; mkdir -p $E
timeout 900 python -m pytest tests/test_gpu_fused_mse.py tests/test_gpu_packed.py tests/test_gpu_window.py -q -x > $E/pytest.log 2>&1; echo "pytest rc=$?" >> $E/pytest.log
tail -n 15 $E/pytest.log
timeout 900 python bench.py --no-cpu-baseline > $E/bench.json 2> $E/bench.err; tail -c 400 $E/bench.json; tail -5 $E/bench.err
