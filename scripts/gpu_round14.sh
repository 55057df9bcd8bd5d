cd $GRAFT_REPO_ROOT/tests
timeout 600 python -m pytest -x -q test_gpu_parity.py -m gpu -k "dense or factorize_matches" 2>&1 | tail -3
cd ..
for div in 100 1000; do
echo "== div $div"
PMMF_B200_DENSE_DIV=$div PMMF_B200_SCORE_TIMING=1 timeout 600 python scripts/three_runs.py 2 > gpurun_out/three_t$div.log 2>&1
grep -E "^run |rror" gpurun_out/three_t$div.log
awk "/^run 0/{f=1} f" gpurun_out/three_t$div.log | grep "score: dense" | head -12 | cut -c1-150
done
