# GPU iteration: parity tests, then one short bench line per config (+ optional ncu case).
set -x
OUT=gpurun_out/${TAG:-it}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo pytest=$?
tail -5 $OUT/pytest.log
for c in ${CONFIGS:-C1 C2 C3 C4 C5}; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2>$OUT/bench_$c.err; echo $c=$?; done
for e in ${EXTRA:-}; do eval "$e"; done
for c in ${CONFIGS:-C1 C2 C3 C4 C5}; do python -c "import json;d=json.load(open('$OUT/bench_$c.json'));print('$c','%.4g'%d['value'],d['ms_per_step'])"; done
