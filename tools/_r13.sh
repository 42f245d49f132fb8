cd $GRAFT_REPO_ROOT
E=gpurun_out/ev2; mkdir -p $E
timeout 300 python tools/probe_host_c2.py > $E/probe_host.log 2>&1; cat $E/probe_host.log | tail -4
timeout 900 python -m pytest tests -x -q -m gpu -k "node or sweep or config2" > $E/t_node.log 2>&1; echo "rc $?" >> $E/t_node.log; tail -n 2 $E/t_node.log
FGFRFT_NODE_PAIRS=1 timeout 900 python -m pytest tests -x -q -m gpu -k "node or sweep or config2" > $E/t_node1.log 2>&1; echo "rc $?" >> $E/t_node1.log; tail -n 2 $E/t_node1.log
timeout 600 python bench.py --no-cpu-baseline > $E/bench_nocpu.json 2>&1; tail -c 600 $E/bench_nocpu.json
