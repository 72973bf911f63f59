#!/bin/bash
# Developer GPU check of a kernel change: the backward parity subset, then bench CONFIGS.
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parallel.py -q -x -k "${TESTK:-backward or fused or autograd or bshd}" > $O/pytest_dev.log 2>&1; tail -3 $O/pytest_dev.log
for c in ${CONFIGS:-cfg2 cfg3}; do
  timeout 300 python bench.py --config $c --no-cpu > $O/bench_dev_$c.log 2>&1
  grep '^{' $O/bench_dev_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), 'fwd', round(d['fwd_ms'],3), 'bwd', d['bwd_ms'] and round(d['bwd_ms'],3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
done
