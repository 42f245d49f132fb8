cd $GRAFT_REPO_ROOT
E=gpurun_out/bands; mkdir -p $E
for nb in 1 0 2 4; do
  FGFRFT_OZ_BANDS=$nb timeout 900 python tools/c3_step.py --config 4 --steps 10 --warmup 3 > $E/c4_b$nb.json 2> $E/c4_b$nb.err
  echo "bands=$nb $(cut -c1-420 $E/c4_b$nb.json)"
done
for nb in 1 2; do
  FGFRFT_OZ_BANDS=$nb timeout 900 python tools/c3_step.py --steps 20 --warmup 4 > $E/c3_b$nb.json 2> $E/c3_b$nb.err
  echo "c3 bands=$nb $(cut -c1-420 $E/c3_b$nb.json)"
done
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_pshard.py tests/test_gpu_fused_mse.py tests/test_gpu_int8gemm.py -m gpu -q -x > $E/pytest.log 2>&1; tail -3 $E/pytest.log
