O=gpurun_out; TAG=${TAG:-r01g}
timeout 900 ncu --set full --clock-control none --import-source on -c 8 -k regex:"mla_" -o $O/prof_cfg4a_${TAG} -f python bench.py --config cfg4a --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -c 8 -k regex:"linear_" -o $O/prof_cfg5a_${TAG} -f python bench.py --config cfg5a --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -c 8 -k regex:"linear_" -o $O/prof_cfg5b_${TAG} -f python bench.py --config cfg5b --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
ls -la $O | grep $TAG
for c in cfg4a cfg5a cfg5b; do python tools/ncu_summary.py $O/prof_${c}_${TAG}.ncu-rep > $O/ncu_summary_${TAG}_${c}.json; done
rm -f $O/prof_cfg5a_${TAG}.ncu-rep $O/prof_cfg5b_${TAG}.ncu-rep
