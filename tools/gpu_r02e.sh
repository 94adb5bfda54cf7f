OUT=gpurun_out/r02e
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CWC_PARITY_OUT=$OUT/parity timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
PROBE_R=16384 python tools/c2_probe.py 10.0 > $OUT/c2_full_probe.jsonl 2>&1; echo probe=$?
