mkdir -p gpurun_out
for G in 14 28 49 14 28 49; do
  v=$(SLB_GROUP2=$G python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['reasons'])")
  echo "G2=$G $v" | tee -a gpurun_out/g2ab2.log
done
