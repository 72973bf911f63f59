#!/bin/bash
# One GPU call: parity suite, smoke, bench of every config (TAG names the outputs).
TAG=${TAG:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu_${TAG}.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $O/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> $O/pytest_${TAG}.log
tail -5 $O/pytest_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_${TAG}.log 2>&1; tail -2 $O/smoke_${TAG}.log
timeout 1800 python bench.py --config all > $O/bench_${TAG}_all.log 2>&1
grep '^{' $O/bench_${TAG}_all.log > $O/bench_${TAG}_all.jsonl
python - <<'PY'
import json,os
tag=os.environ.get("TAG","r02")
for l in open(f"gpurun_out/bench_{tag}_all.jsonl"):
    d=json.loads(l); r=d.get("roofline",{})
    print(d["config"].get("workload","?")[:40], d["value"], d["unit"], d.get("ms_per_step"), "e2e", d.get("e2e",{}).get("value"), "frac", r.get("frac"))
PY
