set -x
OUT=gpurun_out/r02b
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_drawmath.py -q -x > $OUT/pytest_draw.log 2>&1; echo draw=$?
for c in C2 C1 C3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo $c=$?; done
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
