OUT=gpurun_out/r02g
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_resume.py -q -x -k "warp or trace or stall or overflow or no_rules or shard or modes" > $OUT/pytest_warp.log 2>&1; echo pytest=$?
for lib in libcwcsim libcwcsim_oldwarp; do
  L=paper_1010_2438_b200/$lib.so
  python tools/kprobe.py --config C4 --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C5 --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
done
