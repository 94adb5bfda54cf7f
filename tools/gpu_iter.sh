set -x
mkdir -p gpurun_out/r5
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r5/pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r5/pytest.log
for c in C1 C2 C3 C4 C5; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r5/bench_$c.json 2>gpurun_out/r5/bench_$c.err; echo $c=$?; done
python tools/run_case.py --config C2 --t-end 2.0 > gpurun_out/r5/case_C2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:ssa_ -c 1 -o gpurun_out/r5/full_C2 python tools/run_case.py --config C2 --t-end 2.0 > gpurun_out/r5/ncu_C2.log 2>&1; echo ncu=$?
