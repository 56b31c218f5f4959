# A/B of the host batch path with / without lock-step frame pairs (e2e probe, 3 rounds)
for r in 1 2 3; do for v in 0 1; do
  SLB_LOCKSTEP_HOST=$v timeout 120 python tools/e2e_probe.py 8 > /tmp/e2e_$v.txt 2>&1
  echo "host_lockstep=$v $(head -1 /tmp/e2e_$v.txt)"
done; done
