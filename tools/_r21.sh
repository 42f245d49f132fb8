cd $GRAFT_REPO_ROOT
E=gpurun_out/ev3; mkdir -p $E
FGFRFT_NODE_PAIRS=1 timeout 900 python -m pytest tests -x -q -m gpu -k "node or sweep or config2" > $E/t_np.log 2>&1; echo "rc $?" >> $E/t_np.log; tail -n 12 $E/t_np.log
FGFRFT_NODE_PAIRS=1 timeout 300 python tools/probe_regress.py c2 > $E/probe_np.log 2>&1; cut -c1-300 $E/probe_np.log
timeout 300 python tools/probe_regress.py c2 > $E/probe_ne.log 2>&1; cut -c1-300 $E/probe_ne.log
FGFRFT_NODE_PAIRS=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:ozgemm_kernel<\(int\)6, \(int\)0" -s 4 -c 1 -o $E/prof_np python tools/probe_regress.py c2 > $E/ncu_np.log 2>&1
