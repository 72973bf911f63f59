#!/bin/bash
# Round-2 evidence on one GPU box (TAG names the files): the cfg2 launch list and one --set full
# capture per config step (tools/run_step_once.py) of the library's own kernels, condensed by
# tools/ncu_summary.py (durations in ms, head SHA recorded).  The .ncu-rep files stay in /tmp on
# the box (gpurun copies back at most 64 MiB); only the summaries land in gpurun_out/.
# CONFIGS limits the configs (default: all); BENCH=1 also prints the bench lines.
TAG=${TAG:-r02}
CONFIGS=${CONFIGS:-"cfg1 cfg2 cfg3 cfg4a cfg4b cfg5a cfg5b"}
O=gpurun_out
R=/tmp/af_ncu
mkdir -p $O $R
if [ "${BENCH:-0}" = 1 ]; then
  timeout 2400 python bench.py --config all > $O/bench_${TAG}_all.log 2>&1
  grep '^{' $O/bench_${TAG}_all.log > $O/bench_${TAG}_all.jsonl
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_${TAG}_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
for c in $CONFIGS; do
  timeout 1200 ncu --set full --clock-control none --kernel-name-base demangled -k regex:'af::' -o $R/prof_${c}_${TAG} -f \
    python tools/run_step_once.py $c > /dev/null 2>&1
  python tools/ncu_summary.py $R/prof_${c}_${TAG}.ncu-rep > $O/ncu_summary_${TAG}_${c}.json
done
ls -la $O | grep $TAG
