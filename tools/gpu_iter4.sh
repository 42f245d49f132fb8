# Iteration run: digit-emitting synthesis -- packed / fused / window / config tests, then the bench.
cd $GRAFT_REPO_ROOT
E=gpurun_out/it4; mkdir -p $E
timeout 900 python -m pytest tests/test_gpu_packed.py tests/test_gpu_fused_mse.py tests/test_gpu_window.py -q -x > $E/pytest.log 2>&1; echo "pytest rc=$?" >> $E/pytest.log
tail -n 15 $E/pytest.log
for v in 1 0; do
FGFRFT_PSYNTH_DIGITS=$v timeout 900 python bench.py --no-cpu-baseline --no-extras > $E/bench_$v.json 2> $E/bench_$v.err
python -c "
import json;d=json.load(open('$E/bench_$v.json'))
print('digits=$v', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e'].get('h2d_copy_only_ms'), d['kernel_classes'], d['parity_check'])" || tail -5 $E/bench_$v.err
done
timeout 1200 python -m pytest tests/test_gpu_configs.py -q -x -k "config3 or config4" > $E/pytest_cfg.log 2>&1; echo "pytest cfg rc=$?" >> $E/pytest_cfg.log
tail -n 5 $E/pytest_cfg.log
