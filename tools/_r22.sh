cd $GRAFT_REPO_ROOT
E=gpurun_out/ev5; mkdir -p $E
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_configs.py -x -q -k "config5 or config4_packed" > $E/t.log 2>&1; echo "rc $?" >> $E/t.log; tail -n 3 $E/t.log
timeout 600 python tools/c3_step.py --config 4 --steps 5 --warmup 2 --window 0,2 > $E/c4win.log 2>&1; cut -c1-600 $E/c4win.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:batch_dlda_tc" -s 2 -c 1 -o $E/prof_c5d python tools/bench_configs.py --configs 5 > $E/ncu_c5d.log 2>&1
