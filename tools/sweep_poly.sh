#!/bin/bash
# Developer ablation: fraction of K1 exponentials evaluated by exp2_poly (FMA pipe) vs MUFU.
for m in ${MASKS:-14 6 2 0}; do
  AF_EXTRA_NVCC_FLAGS="-DAF_EXP2_POLY_MASK=$m" python -c "from paper_2502_15349_b200 import build; build.build_library()" > /dev/null 2>&1
  echo "mask=$m $(python bench.py --config cfg2 --no-cpu --steps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["fwd_tflops"])')"
done
