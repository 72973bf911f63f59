#!/bin/bash
# Developer ablation: MLA prefill latent-tile width (64 x 2 stages vs 32 x 4 stages).
for n in 32 64; do
  AF_EXTRA_NVCC_FLAGS="-DAF_MLA_PREFILL_N=$n" python -c "from paper_2502_15349_b200 import build; build.build_library()" > /dev/null 2>&1
  echo "N=$n"; python tools/probe_mla.py 2>&1 | grep TIME
done
