# A/B of SLB_CHUNK1 (bands per chunk with 1-3 frames in flight) on bench.py 2d512
mkdir -p gpurun_out
for C in default 14 28 default 14 28; do
  if [ "$C" = default ]; then e=""; else e="SLB_CHUNK1=$C"; fi
  v=$(env $e python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['reasons'])")
  echo "CHUNK1=$C $v" | tee -a gpurun_out/chunk1ab.log
done
