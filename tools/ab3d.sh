# A/B the 3D path across prebuilt library variants (paper_1402_5670_b200/libab_<v>.so)
for v in ${VARIANTS:-A}; do
  for c in ${CONFIGS:-3d192}; do
    SLB_LIB=$PWD/paper_1402_5670_b200/libab_$v.so python bench.py --config $c --no-cpu-baseline --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$c', round(d['value'],2), {k: round(v['ms_total']/v['launches'],4) for k,v in d['kernels'].items()})"
  done
done
