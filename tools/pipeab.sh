# A/B of SLB_HOST_PIPE (compute streams of the pipelined host batch) on bench.py 2d512
mkdir -p gpurun_out
for P in 3 2 4 3 2 4; do
  v=$(SLB_HOST_PIPE=$P python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['reasons'])")
  echo "HOST_PIPE=$P $v" | tee -a gpurun_out/pipeab.log
done
