cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev2
E=gpurun_out/ev2
timeout 900 python -m pytest tests -x -q -m gpu -k "node or sweep or config2" > $E/t_node.log 2>&1; echo "rc $?" >> $E/t_node.log; tail -3 $E/t_node.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:ozgemm_kernel<\(int\)6, \(int\)0" -s 4 -c 1 -o $E/prof_nodeop_pairs python tools/probe_regress.py c2 > $E/ncu_np.log 2>&1
FGFRFT_NODE_PAIRS=0 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:ozgemm_kernel<\(int\)6, \(int\)0" -s 4 -c 1 -o $E/prof_nodeop_elem python tools/probe_regress.py c2 > $E/ncu_ne.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:ozgemm_kernel<\(int\)6, \(int\)1|oz_slice_direct_kernel<\(int\)6>|oz_rowslice_pairs_kernel<\(int\)6>" -s 3 -c 3 -o $E/prof_c3g python tools/c3_step.py --steps 2 --warmup 2 > $E/ncu_c3g.log 2>&1
tail -2 $E/ncu_c3g.log $E/ncu_np.log
