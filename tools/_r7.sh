cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/t_batch.log 2>&1; echo "rc $?" >> gpurun_out/t_batch.log
tail -2 gpurun_out/t_batch.log
for st in 8 6 4; do FGFRFT_TC_STAGES=$st timeout 300 python tools/bench_configs.py --configs 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('stages $st', 'fwd', round(d['forward']['ms'],4), 'dlda', round(d['dlda']['ms'],4))"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:batch_fwd_tc -s 2 -c 1 -o gpurun_out/c5fwd3 python tools/bench_configs.py --configs 5 > gpurun_out/ncu_c5.log 2>&1
