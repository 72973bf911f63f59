#!/bin/bash
# Developer ablation on one box: bench CFG with the in-tree library, then rebuilt with the
# developer flags in ABL (e.g. -DAF_FUSED_NO_REDUCE), then restored.
CFG=${CFG:-cfg2}
O=gpurun_out; mkdir -p $O
run() { timeout 300 python bench.py --config $CFG --no-cpu --steps 10 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["value"])'; }
echo "base   $(run)"
AF_EXTRA_NVCC_FLAGS="$ABL" python -c "from paper_2502_15349_b200 import build; build.build_library()" > /dev/null 2>&1
echo "ablate($ABL) $(run)"
python -c "from paper_2502_15349_b200 import build; build.build_library()" > /dev/null 2>&1
echo "base   $(run)"
