#!/bin/bash
# Developer ablation: fraction of the K2a/K2b P-recompute exponentials on the FMA pipe.
for m in ${MASKS:--1 14 6}; do
  AF_EXTRA_NVCC_FLAGS="-DAF_BWD_POLY_MASK=$m" python -c "from paper_2502_15349_b200 import build; build.build_library()" > /dev/null 2>&1
  echo "mask=$m $(python bench.py --config cfg2 --no-cpu --steps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["bwd_ms"], d["bwd_tflops"])')"
done
