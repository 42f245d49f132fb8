cd $GRAFT_REPO_ROOT
E=gpurun_out/ev2; mkdir -p $E
timeout 300 python tools/probe_host_c2.py > $E/probe_host.log 2>&1; cat $E/probe_host.log | tail -5
FGFRFT_NODE_PAIRS=0 timeout 300 python tools/probe_host_c2.py > $E/probe_host0.log 2>&1; cat $E/probe_host0.log | tail -5
nproc; cat /proc/loadavg
