#!/bin/bash
# Developer ablation over nvcc -D flag sets (one per argument), alternating twice on one box:
#   CFG=cfg2 bash tools/sweep_flags.sh "-DAF_FWD_PACK=0" "-DAF_FWD_PACK=2"
CFG=${CFG:-cfg2}
for round in 1 2; do
  for f in "$@"; do
    AF_EXTRA_NVCC_FLAGS="$f" python -c "from paper_2502_15349_b200 import build; build.build_library()" > /dev/null 2>&1
    echo "[$f] $(python bench.py --config $CFG --no-cpu --steps 10 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d.get("bwd_ms"), d["value"])')"
  done
done
