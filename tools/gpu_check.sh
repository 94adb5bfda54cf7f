# GPU check: parity tests, smoke, one short bench line per config (one GPU).
set -x
OUT=gpurun_out/check
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
for c in ${CONFIGS:-C1 C2 C3 C4 C5}; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo $c=$?
done
cat $OUT/bench_*.json
