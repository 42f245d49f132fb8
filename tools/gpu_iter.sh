# One build -> measure iteration on the GPU box: GPU tests (optionally filtered by $K), the bench
# and its ncu launch list, under gpurun_out/r1/.
mkdir -p gpurun_out/r1
python -m pytest tests -m gpu -q -x ${K:+-k "$K"} > gpurun_out/r1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1/pytest.log
python bench.py --no-cpu-baseline > gpurun_out/r1/bench.json 2> gpurun_out/r1/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
tail -2 gpurun_out/r1/pytest.log
