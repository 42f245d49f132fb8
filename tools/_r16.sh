cd $GRAFT_REPO_ROOT
E=gpurun_out/ev2; mkdir -p $E
timeout 900 python -m pytest tests/test_gpu_window.py -x -q > $E/t_win.log 2>&1; echo "rc $?" >> $E/t_win.log; tail -n 3 $E/t_win.log
timeout 300 python tools/c3_step.py --steps 10 --warmup 3 --window 0,2 > $E/c3win.log 2>&1; cut -c1-600 $E/c3win.log
timeout 300 python tools/c3_step.py --steps 10 --warmup 3 --window 0.25,0.75 > $E/c3win2.log 2>&1; cut -c1-600 $E/c3win2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:window_synth -s 2 -c 1 -o $E/prof_win2 python tools/c3_step.py --steps 2 --warmup 2 --window 0,2 > $E/ncu_win.log 2>&1
