cd $GRAFT_REPO_ROOT
cd tests && timeout 900 python -m pytest -x -q test_gpu_parity.py -m gpu -k "cluster_search or c2_rmat or rmat14" 2>&1 | tail -2; cd ..
PMMF_B200_TRACE=1 timeout 600 python scripts/configs_full.py c5 --no-pcg > gpurun_out/c5b.log 2> gpurun_out/c5b.err; echo rc=$?
cat gpurun_out/c5b.log | cut -c1-300; grep -E "stage [1-3]: (search)|search:" gpurun_out/c5b.err | head -8
timeout 600 python scripts/three_runs.py 2 > gpurun_out/c4t.log 2>&1; grep -E "^run" gpurun_out/c4t.log
grep -E "search:|apply\.|stage [0-9]+: (gram|apply)|batch cols|masses" gpurun_out/c4t.log | sed -n '/run 1/,$p' | head -5
sed -n '/^run 0/,$p' gpurun_out/c4t.log | grep -E "search:|apply\.|stage [0-9]+: (gram|apply|wall)" | head -60
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_stage_apply_k -c 2 -o gpurun_out/prof_apply python scripts/configs_full.py c5 --no-pcg --apply-only > gpurun_out/ncu_apply.log 2>&1; tail -2 gpurun_out/ncu_apply.log
