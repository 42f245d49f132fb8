# A/B of the fused MSE on the bench (device step) and the e2e variance check.
cd $GRAFT_REPO_ROOT
E=gpurun_out/it3; mkdir -p $E
for v in 1 0 1; do
FGFRFT_FUSED_MSE=$v timeout 900 python bench.py --no-cpu-baseline --no-extras > $E/bench_$v.json 2> $E/bench_$v.err
python -c "
import json;d=json.load(open('$E/bench_$v.json'))
print('fused=$v', d['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_classes']['elementwise']['ms_per_step'], d['kernel_classes']['int8_gemm']['ms_per_step'])"
done
