# A/B the 2D headline path across prebuilt library variants (paper_1402_5670_b200/libab_<v>.so)
for v in ${VARIANTS:-A}; do
  SLB_LIB=$PWD/paper_1402_5670_b200/libab_$v.so python bench.py --no-3d --no-cpu-baseline --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['e2e']['value']), {k: round(v['ms_total']/v['bands']*1000,3) for k,v in d['kernels'].items() if v['bands']>100})"
done
