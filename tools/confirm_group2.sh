cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do for g in 7 ""; do echo "[SLB_GROUP2=${g:-default}] $(env ${g:+SLB_GROUP2=$g} timeout 120 python tools/e2e_probe.py 8 2>&1 | head -1)"; done; done
python bench.py --steps 50 --warmup 3 > gpurun_out/bench_r1q.json 2> gpurun_out/bench_r1q.err; tail -c 600 gpurun_out/bench_r1q.json
