# Addendum to the round-end evidence: ncu --set full of each config's SSA kernel at the bench workload,
# summarised with the pipe mix and the derived issue / SIMT / divergence fractions (tools/ncu_summary.py)
OUT=gpurun_out/pipes
mkdir -p $OUT
for c in C2 C3 C4 C5; do
  python tools/run_case.py --config $c > $OUT/case_$c.log 2>&1 && \
  ncu --set full --clock-control none -k regex:ssa_ -c 1 -o $OUT/full_$c python tools/run_case.py --config $c > $OUT/ncu_$c.log 2>&1
  echo $c=$?
done
python tools/ncu_summary.py $OUT/ncu_pipe_summary.json $(for c in C2 C3 C4 C5; do [ -f $OUT/full_$c.ncu-rep ] && echo $c=$OUT/full_$c.ncu-rep; done) > $OUT/ncu_pipe_summary.log 2>&1; echo summary=$?
ncu -i $OUT/full_C4.ncu-rep --page raw --csv 2>/dev/null | head -1 | tr ',' '\n' | grep -c "inst_executed_pipe"
rm -f $OUT/full_*.ncu-rep
