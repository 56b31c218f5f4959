cd $GRAFT_REPO_ROOT
SLB_LIB=$PWD/paper_1402_5670_b200/libab_direct.so timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do VARIANTS="base direct" bash tools/ab_libs.sh; done
for c in 3d192 3d128 2d1024x64; do for v in base direct; do
  SLB_LIB=$PWD/paper_1402_5670_b200/libab_$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$c', round(d['value'],2), round(d['e2e']['value'],2), {k: round(v['ms_total']/v['launches'],4) for k,v in d['kernels'].items() if 'rows' in k})"
done; done
