#!/bin/bash
# Round-end evidence on one GPU box: bench lines for every config (with the CPU baseline), the
# cfg2 launch list, and --set full captures of the dominant kernels.  TAG names the files.
TAG=${TAG:-r01g}
O=gpurun_out
mkdir -p $O
timeout 1500 python bench.py --config all > $O/bench_${TAG}_all.log 2>&1
grep '^{' $O/bench_${TAG}_all.log > $O/bench_${TAG}_all.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_${TAG}_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"parallel_(fwd|bwd_dkdv|bwd_dq)_kernel" -c 3 -o $O/prof_cfg2_${TAG} -f \
  python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"parallel_(fwd|bwd_dkdv|bwd_dq)_kernel" -c 3 -o $O/prof_cfg3_${TAG} -f \
  python bench.py --config cfg3 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"mla_" -c 2 -o $O/prof_cfg4b_${TAG} -f \
  python bench.py --config cfg4b --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
ls -la $O | grep $TAG
