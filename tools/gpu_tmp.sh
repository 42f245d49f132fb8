cd $GRAFT_REPO_ROOT
E=gpurun_out/e2e; mkdir -p $E
PROBE_DS=0 timeout 600 python tools/probe_regress.py c3 > $E/c3_a.jsonl 2>&1
PROBE_DS=0 FGFRFT_PSYNTH_DIGITS=0 timeout 600 python tools/probe_regress.py c3 > $E/c3_b.jsonl 2>&1
cut -c1-400 $E/c3_a.jsonl; cut -c1-400 $E/c3_b.jsonl
timeout 900 python bench.py --no-cpu-baseline --no-extras > $E/bench.json 2> $E/bench.err
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/e2e/bench.json') if l.startswith('{')][-1])
print(d['ms_per_step'], d['e2e'])
PY
