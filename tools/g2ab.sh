# A/B of SLB_GROUP2 (2D band group with 2-3 frames in flight) on bench.py 2d512; G2LIST overrides the list
mkdir -p gpurun_out
for G in ${G2LIST:-14 28 49 14 28 49}; do
  v=$(SLB_GROUP2=$G python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['reasons'])")
  echo "G2=$G $v" | tee -a gpurun_out/g2ab2.log
done
