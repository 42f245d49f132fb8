cd $GRAFT_REPO_ROOT
E=gpurun_out/dq; mkdir -p $E
timeout 600 python tools/c3_step.py --steps 20 --warmup 4 --sweep 'FGFRFT_DQ_DIGITS=6;FGFRFT_DQ_DIGITS=5;FGFRFT_DQ_DIGITS=4;FGFRFT_DQ_DIGITS=6;FGFRFT_DQ_DIGITS=5' > $E/c3.jsonl 2> $E/c3.err
timeout 600 python tools/c3_step.py --steps 21 --warmup 4 --sweep 'FGFRFT_DQ_DIGITS=6;FGFRFT_DQ_DIGITS=5;FGFRFT_DQ_DIGITS=4' > $E/c3_odd.jsonl 2> $E/c3_odd.err
timeout 600 python tools/c3_step.py --steps 20 --warmup 4 --window 0,2 --sweep 'FGFRFT_DQ_DIGITS=6;FGFRFT_DQ_DIGITS=5;FGFRFT_DQ_DIGITS=4' > $E/c3_win.jsonl 2> $E/c3_win.err
timeout 900 python tools/c3_step.py --config 4 --steps 10 --warmup 3 --sweep 'FGFRFT_DQ_DIGITS=6;FGFRFT_DQ_DIGITS=5;FGFRFT_DQ_DIGITS=4' > $E/c4.jsonl 2> $E/c4.err
FGFRFT_DQ_DIGITS=5 timeout 900 python -m pytest tests/test_gpu_packed.py tests/test_gpu_window.py tests/test_gpu_configs.py -m gpu -q -x > $E/pytest5.log 2>&1; tail -3 $E/pytest5.log
cat $E/c3.jsonl $E/c3_odd.jsonl $E/c3_win.jsonl $E/c4.jsonl | cut -c1-400
