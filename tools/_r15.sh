cd $GRAFT_REPO_ROOT
E=gpurun_out/ev2; mkdir -p $E
FGFRFT_HOST_PROF=1 timeout 600 python tools/probe_host_c2.py > $E/probe_host.log 2>&1; cat $E/probe_host.log | tail -12
timeout 900 python -m pytest tests/test_gpu_window.py -x -q > $E/t_win.log 2>&1; echo "rc $?" >> $E/t_win.log; tail -n 15 $E/t_win.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:window_synth -s 2 -c 1 -o $E/prof_win python tools/c3_step.py --steps 2 --warmup 2 --window 0,2 > $E/ncu_win.log 2>&1
tail -n 2 $E/ncu_win.log
