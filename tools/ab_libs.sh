for v in ${VARIANTS:-680a406 cur}; do
  SLB_LIB=$PWD/paper_1402_5670_b200/libab_$v.so python bench.py --no-cpu-baseline --steps 30 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['e2e']['value']), {k: round(v['ms_total']/v['launches'],4) for k,v in d['kernels'].items()})"
done
