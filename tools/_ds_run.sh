cd $GRAFT_REPO_ROOT
SW="FGFRFT_DSYNTH=1"
for sp in "0.3" "0.4" "0.25,0.5" "0.3,0.6" "0.2,0.4,0.6"; do for gc in 80; do SW="$SW;FGFRFT_PIPE_SPLIT=$sp&FGFRFT_PIPE_GEMM_CTAS=$gc"; done; done
timeout 900 python tools/c3_step.py --steps 5 --warmup 3 --trace --sweep "$SW" 2>&1 | tail -12 | cut -c1-1500
