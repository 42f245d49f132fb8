cd $GRAFT_REPO_ROOT
E=gpurun_out/ev7; mkdir -p $E
for pf in 1 0; do FGFRFT_TC_PREFETCH=$pf timeout 300 python tools/bench_configs.py --configs 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('prefetch $pf', 'fwd', round(d['forward']['ms'],4), 'dlda', round(d['dlda']['ms'],4))"; done
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > $E/t_batch.log 2>&1; echo "rc $?" >> $E/t_batch.log; tail -n 2 $E/t_batch.log
