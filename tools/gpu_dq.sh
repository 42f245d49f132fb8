cd $GRAFT_REPO_ROOT
E=gpurun_out/pb; mkdir -p $E
timeout 900 python -m pytest tests/test_gpu_packed.py tests/test_gpu_window.py tests/test_gpu_configs.py tests/test_gpu_pshard.py tests/test_gpu_fused_mse.py -m gpu -q -x > $E/pytest.log 2>&1; tail -3 $E/pytest.log
timeout 600 python tools/c3_step.py --steps 20 --warmup 4 > $E/c3.jsonl 2> $E/c3.err
timeout 600 python tools/c3_step.py --steps 20 --warmup 4 >> $E/c3.jsonl 2>> $E/c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $E/launches.csv python tools/c3_step.py --steps 2 --warmup 2 > $E/ncu.log 2>&1
cat $E/c3.jsonl | cut -c1-600
grep -E "prow_bound|fused_mse_finish" $E/launches.csv | tail -4 | cut -c1-300
