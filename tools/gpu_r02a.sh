set -x
OUT=gpurun_out/r02a
mkdir -p $OUT
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
./tools/pipebench/pipe_bench > $OUT/pipe_bench.json 2> $OUT/pipe_bench.err; echo pipe=$?
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo bench=$?
for c in C3 C4 C5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo $c=$?; done
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
