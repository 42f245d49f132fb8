cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev2
E=gpurun_out/ev2
timeout 900 python -m pytest tests -x -q -m gpu -k "node or sweep or config2" > $E/t_node.log 2>&1; echo "rc $?" >> $E/t_node.log; tail -3 $E/t_node.log
timeout 300 python tools/probe_regress.py c2 > $E/probe_pairs.log 2>&1
FGFRFT_NODE_PAIRS=0 timeout 300 python tools/probe_regress.py c2 >> $E/probe_pairs.log 2>&1
cut -c1-300 $E/probe_pairs.log
timeout 600 python tools/probe_c2_after_c3.py > $E/probe_c2.log 2>&1; cut -c1-400 $E/probe_c2.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ozgemm_kernel<6, 1|oz_slice_direct_kernel<6>|oz_rowslice_pairs_kernel<6>" -s 3 -c 3 -o $E/prof_c3g python tools/c3_step.py --steps 2 --warmup 2 > $E/ncu_c3g.log 2>&1
tail -2 $E/ncu_c3g.log
