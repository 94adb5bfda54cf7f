OUT=gpurun_out/r02p
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=8 > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo bench=$?
for c in C1 C3 C4 C5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo $c=$?; done
for c in C2 C4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --dump > $OUT/bench_dump_$c.json 2> $OUT/bench_dump_$c.err; echo dump$c=$?; done
for c in C1 C2 C3 C4 C5; do for m in shared global; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --stats-mode $m > $OUT/bench_stats_${c}_$m.json 2> $OUT/bench_stats_${c}_$m.err; echo stats$c$m=$?; done; done
