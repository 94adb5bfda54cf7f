OUT=gpurun_out/r02f
mkdir -p $OUT
for lib in libcwcsim libcwcsim_tb2 libcwcsim_i2dcvt libcwcsim_logcvt libcwcsim_nowide; do
  L=paper_1010_2438_b200/$lib.so
  python tools/kprobe.py --config C2 --t-end 2 --kernel single --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C2 --t-end 2 --kernel ws --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C2 --t-end 2 --kernel single --replicas 32 --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C3 --kernel single --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C1 --kernel ws --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
done
