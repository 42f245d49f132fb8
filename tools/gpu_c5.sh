mkdir -p gpurun_out/c5
python -m pytest tests -m gpu -q -x -k "batch" > gpurun_out/c5/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c5/pytest.log
python tools/bench_configs.py --configs 5 > gpurun_out/c5/c5.jsonl 2> gpurun_out/c5/c5.err
tail -2 gpurun_out/c5/pytest.log
