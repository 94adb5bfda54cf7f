# Pipe mix of the warp kernels (ncu --set full, shortened horizons), summarised by tools/ncu_summary.py
OUT=gpurun_out/pipes2
mkdir -p $OUT
python tools/run_case.py --config C4 --t-end 0.3 > $OUT/case_C4.log 2>&1 && ncu --set full --clock-control none -k regex:ssa_ -c 1 -o $OUT/full_C4 python tools/run_case.py --config C4 --t-end 0.3 > $OUT/ncu_C4.log 2>&1; echo C4=$?
python tools/run_case.py --config C5 --t-end 5 > $OUT/case_C5.log 2>&1 && ncu --set full --clock-control none -k regex:ssa_ -c 1 -o $OUT/full_C5 python tools/run_case.py --config C5 --t-end 5 > $OUT/ncu_C5.log 2>&1; echo C5=$?
python tools/run_case.py --config C2 --t-end 2 > $OUT/case_C2.log 2>&1 && ncu --set full --clock-control none -k regex:ssa_ -c 1 -o $OUT/full_C2 python tools/run_case.py --config C2 --t-end 2 > $OUT/ncu_C2.log 2>&1; echo C2=$?
python tools/ncu_summary.py $OUT/ncu_pipe_summary.json C4=$OUT/full_C4.ncu-rep C5=$OUT/full_C5.ncu-rep C2=$OUT/full_C2.ncu-rep > $OUT/ncu_pipe_summary.log 2>&1; echo summary=$?
ncu -i $OUT/full_C4.ncu-rep --page raw --csv 2>/dev/null | head -1 | tr ',' '\n' | grep "inst_executed_pipe" | head -100 > $OUT/pipe_metric_names.txt
rm -f $OUT/full_*.ncu-rep
python -c "
import json
s=json.load(open('$OUT/ncu_pipe_summary.json'))
for c,v in s.items(): print(c, v.get('pipe_util_pct'))
"
