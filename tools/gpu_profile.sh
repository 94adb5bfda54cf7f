# ncu evidence for the bench command and the two SSA kernels (one GPU).
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --steps 2 --warmup 3 > $OUT/bench_plain.json 2> $OUT/bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 > $OUT/bench_ncu.log 2>&1
echo launches=$?
for c in C2 C4 C5 C3; do
  python tools/run_case.py --config $c > $OUT/case_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ssa_ -c 1 -o $OUT/full_$c \
      python tools/run_case.py --config $c > $OUT/ncu_$c.log 2>&1
  echo $c=$?
done
ls -la $OUT
