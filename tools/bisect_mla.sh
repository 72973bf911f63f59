#!/bin/bash
# Developer bisect: the MLA determinism probe against the working tree and against staged
# variants of the MLA sources in .bisect/ (each rebuilt in turn).
run() { timeout 300 python tools/probe_mla_determinism.py 2>&1 | tail -1; }
echo "== working tree"; run
for v in .bisect/variant_*; do
  [ -d "$v" ] || continue
  cp "$v"/* paper_2502_15349_b200/csrc/
  python -c "from paper_2502_15349_b200 import build; build.build_library()" > /dev/null 2>&1
  echo "== $v"; run
done
