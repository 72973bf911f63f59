#!/bin/bash
# Developer A/B on one box: bench the working tree (B), then the files staged under
# .ab_old/ swapped into csrc/ (A), alternating, so box-to-box variance cancels.
CFG=${CFG:-cfg2}
run() { python bench.py --config $CFG --no-cpu --steps 10 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["value"])'; }
mkdir -p /tmp/ab_new && cp paper_2502_15349_b200/csrc/* /tmp/ab_new/
for round in 1 2; do
  cp /tmp/ab_new/* paper_2502_15349_b200/csrc/; python -c "from paper_2502_15349_b200 import build; build.build_library()" >/dev/null 2>&1
  echo "B(new) $(run)"
  cp .ab_old/* paper_2502_15349_b200/csrc/; python -c "from paper_2502_15349_b200 import build; build.build_library()" >/dev/null 2>&1
  echo "A(old) $(run)"
done
cp /tmp/ab_new/* paper_2502_15349_b200/csrc/
