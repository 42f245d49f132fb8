cd $GRAFT_REPO_ROOT
E=gpurun_out/ev3; mkdir -p $E
timeout 900 python -m pytest tests -x -q -m gpu -k "node or sweep or config2 or window or synth or sinc" > $E/t_node.log 2>&1; echo "rc $?" >> $E/t_node.log; tail -n 2 $E/t_node.log
FGFRFT_HOST_PROF=1 timeout 900 python bench.py --no-cpu-baseline > $E/bench_hp.json 2> $E/bench_hp.err
python -c "
import json; d=json.loads(open('$E/bench_hp.json').read().strip().splitlines()[-1]); print('c2', d['c2_sweep']['ms_per_step'], 'c3', d['ms_per_step'], 'win', d['order_window_step']['ms_per_step'])"
grep "fgfrft host" $E/bench_hp.err
