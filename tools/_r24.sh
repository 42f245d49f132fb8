cd $GRAFT_REPO_ROOT
E=gpurun_out/ev5; mkdir -p $E
timeout 300 python tools/probe_regress.py c2 > $E/probe_c2.log 2>&1; cut -c1-300 $E/probe_c2.log
FGFRFT_NODE_PAIRS=1 timeout 300 python tools/probe_regress.py c2 > $E/probe_c2p.log 2>&1; cut -c1-300 $E/probe_c2p.log | head -1
timeout 900 python -m pytest tests -x -q -m gpu -k "node or sweep or config2 or int8" > $E/t_node.log 2>&1; echo "rc $?" >> $E/t_node.log; tail -n 2 $E/t_node.log
FGFRFT_NODE_PAIRS=1 timeout 900 python -m pytest tests -x -q -m gpu -k "node or sweep or config2" > $E/t_node1.log 2>&1; echo "rc $?" >> $E/t_node1.log; tail -n 2 $E/t_node1.log
