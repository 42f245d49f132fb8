cd $GRAFT_REPO_ROOT
E=gpurun_out/ev3; mkdir -p $E
FGFRFT_HOST_PROF=1 timeout 900 python bench.py --no-cpu-baseline > $E/bench_hp.json 2> $E/bench_hp.err
python -c "
import json; d=json.loads(open('$E/bench_hp.json').read().strip().splitlines()[-1]); print('c2', d['c2_sweep']['ms_per_step'])"
grep "fgfrft host" $E/bench_hp.err
OMP_WAIT_POLICY=passive FGFRFT_HOST_PROF=1 timeout 900 python bench.py --no-cpu-baseline > $E/bench_hp2.json 2> $E/bench_hp2.err
python -c "
import json; d=json.loads(open('$E/bench_hp2.json').read().strip().splitlines()[-1]); print('c2 passive', d['c2_sweep']['ms_per_step'])"
grep "fgfrft host" $E/bench_hp2.err
