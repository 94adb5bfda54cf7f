# Round evidence: GPU tests, smoke, bench lines (all configs), the ncu launch
# list of the default bench command, and one ncu --set full capture of the
# SSA kernel at each config's bench workload (for `traffic` and counters).
set -x
OUT=gpurun_out/${TAG:-final}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo bench=$?
for c in C1 C2 C3 C4 C5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo $c=$?; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo ref=$?
# the dynamic-topology workload (NEXT-4) and its oracle arm
timeout 600 python bench.py --config C6 --steps 5 --warmup 3 > $OUT/bench_C6.json 2> $OUT/bench_C6.err; echo C6=$?
timeout 300 python bench.py --config C6 --impl reference --steps 2 --warmup 1 > $OUT/bench_C6_reference.json 2> $OUT/bench_C6_reference.err; echo C6ref=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/launch_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/launch_ncu.log 2>&1; echo launches=$?
for c in ${FULLCASES:-C2 C1 C3 C4 C5}; do
  python tools/run_case.py --config $c > $OUT/case_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ssa_ -c 1 -o $OUT/full_$c \
      python tools/run_case.py --config $c > $OUT/ncu_$c.log 2>&1; echo full_$c=$?
done
python tools/dyn_probe.py 8192 > $OUT/case_C6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dyn_ -c 1 -o $OUT/full_C6 \
    python tools/dyn_probe.py 8192 > $OUT/ncu_C6.log 2>&1; echo full_C6=$?
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB return limit):
# counters per config, per-source-line tables, and only the default config's report
python tools/ncu_summary.py $OUT/ncu_full_summary.json $(for c in ${FULLCASES:-C2 C1 C3 C4 C5} C6; do [ -f $OUT/full_$c.ncu-rep ] && echo $c=$OUT/full_$c.ncu-rep; done) > $OUT/ncu_summary.log 2>&1; echo summary=$?
for c in ${FULLCASES:-C2 C1 C3 C4 C5} C6; do [ -f $OUT/full_$c.ncu-rep ] && python tools/ncu_lines.py $OUT/full_$c.ncu-rep 60 > $OUT/lines_$c.txt 2>&1; done
# parity reports (survey subsets, every trajectory of the five configs, C6)
if [ -n "$PARITY" ]; then
  CWC_PARITY_OUT=$OUT/parity_scale timeout 1200 python -m pytest tests/test_gpu_parity_scale.py -q > $OUT/parity_scale.log 2>&1; echo parity_scale=$?
  CWC_PARITY_FULL=1 CWC_PARITY_OUT=$OUT/parity_full timeout 2400 python -m pytest tests/test_gpu_parity_full.py -q > $OUT/parity_full.log 2>&1; echo parity_full=$?
  CWC_PARITY_OUT=$OUT/parity_dyn timeout 900 python -m pytest tests/test_gpu_dynamic.py -q -k survey > $OUT/parity_dyn.log 2>&1; echo parity_dyn=$?
fi
# dump mode: DRAM bytes of the SSA kernel with and without the trajectory dump (write amplification)
for c in C2 C4; do
  python tools/run_case.py --config $c --t-end ${DUMP_T:-0.5} --dump > $OUT/dumpcase_$c.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ssa_ -c 1 --csv \
      --log-file $OUT/dump_dram_$c.csv python tools/run_case.py --config $c --t-end ${DUMP_T:-0.5} --dump > $OUT/dumpncu_$c.log 2>&1; echo dump_$c=$?
  python tools/run_case.py --config $c --t-end ${DUMP_T:-0.5} > $OUT/nodumpcase_$c.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ssa_ -c 1 --csv \
      --log-file $OUT/nodump_dram_$c.csv python tools/run_case.py --config $c --t-end ${DUMP_T:-0.5} > $OUT/nodumpncu_$c.log 2>&1; echo nodump_$c=$?
done
mkdir -p $OUT/../reps_${TAG:-final}
for c in ${FULLCASES:-C2 C1 C3 C4 C5} C6; do rm -f $OUT/full_$c.ncu-rep; done
