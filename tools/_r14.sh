cd $GRAFT_REPO_ROOT
E=gpurun_out/ev2; mkdir -p $E
timeout 900 python -m pytest tests/test_gpu_window.py -x -q > $E/t_win.log 2>&1; echo "rc $?" >> $E/t_win.log; tail -n 15 $E/t_win.log
timeout 300 python tools/c3_step.py --steps 10 --warmup 3 --window 0,2 > $E/c3win.log 2>&1; cut -c1-700 $E/c3win.log
timeout 300 python tools/c3_step.py --steps 10 --warmup 3 > $E/c3.log 2>&1; cut -c1-500 $E/c3.log
timeout 600 python tools/probe_host_c2.py > $E/probe_host.log 2>&1; cat $E/probe_host.log | tail -4
