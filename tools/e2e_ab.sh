# A/B of a host batch path knob with the e2e probe, 3 rounds: VAR in {A, B} values
VAR=${VAR:-SLB_HOST_PRIO}; A=${A:-0}; B=${B:-1}
for r in 1 2 3; do for v in $A $B; do
  env $VAR=$v timeout 120 python tools/e2e_probe.py 8 > /tmp/e2e_$v.txt 2>&1
  echo "$VAR=$v $(head -2 /tmp/e2e_$v.txt | tr '\n' ' ')"
done; done
