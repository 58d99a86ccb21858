#!/bin/bash
# A/B of gather knobs on one box (alternating rounds): prints value / e2e /
# single-batch call per variant. Usage: bash tools/diag/ab_gather.sh "ENV=.. ENV=.." "ENV=.." ...
# (an empty string is the default build). Output: gpurun_out/ab_gather.txt
out=gpurun_out/ab_gather.txt
mkdir -p gpurun_out
: > $out
for round in 1 2; do
  for v in "$@"; do
    line=$(env $v timeout 300 python bench.py --no-sgd --no-c3 --no-c4 --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | tail -1)
    python - "$v" "$line" >> $out <<'EOF'
import json, sys
v, line = sys.argv[1], sys.argv[2]
try:
    j = json.loads(line)
    sb = j["e2e"].get("single_batch_call", {})
    print("round variant=%-40s value %7.1f  e2e %7.1f  frac %.4f  single_us %.2f  sm %s" % (
        v or "default", j["value"], j["e2e"]["value"], j["roofline"]["frac"], sb.get("us_per_call", -1),
        j.get("clocks", {}).get("sm_mhz")))
except Exception as e:
    print("variant=%s failed: %s %s" % (v, e, line[:200]))
EOF
  done
done
cat $out
