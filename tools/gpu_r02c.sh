OUT=gpurun_out/r02c
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python tools/c2_probe.py 2.0 > $OUT/c2_probe.jsonl 2> $OUT/c2_probe.err; echo probe=$?
python tools/run_case.py --config C2 --t-end 2 > $OUT/case.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ssa_ -c 1 -o $OUT/c2full python tools/run_case.py --config C2 --t-end 2 > $OUT/ncu.log 2>&1; echo ncu=$?
python tools/ncu_lines.py $OUT/c2full.ncu-rep 80 > $OUT/lines_C2.txt 2>&1
python tools/ncu_summary.py $OUT/ncu_sum.json C2=$OUT/c2full.ncu-rep > $OUT/sum.log 2>&1
