# ncu --set full of the SSA kernel on selected configs: CASES="C2:2.0 C3:" (config:t_end)
set -x
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
for cs in ${CASES:-C2:2.0}; do
  c=${cs%%:*}; te=${cs#*:}; arg=""; [ -n "$te" ] && arg="--t-end $te"
  python tools/run_case.py --config $c $arg > $OUT/case_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ssa_ -c 1 -o $OUT/full_$c \
      python tools/run_case.py --config $c $arg > $OUT/ncu_$c.log 2>&1
  echo $c=$?
done
