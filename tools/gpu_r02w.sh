# A/B of the predicated-shuffle scan steps (libcwcsim_scan.so) against the
# committed build (libcwcsim.so): C4, C5 kernel times and the group-kernel crossover
OUT=gpurun_out/scan
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
for lib in libcwcsim.so libcwcsim_scan.so libcwcsim_scan2.so; do
  for c in C4 C5; do
    python tools/kprobe.py --config $c --lib paper_1010_2438_b200/$lib >> $OUT/kprobe.jsonl 2>> $OUT/err.log
  done
  CWC_PROBE_LIB=paper_1010_2438_b200/$lib python tools/dyn_probe.py 8192 | tail -1 | sed "s/^/$lib /" >> $OUT/dyn.txt 2>> $OUT/err.log
  python tools/warp8_crossover.py paper_1010_2438_b200/$lib >> $OUT/crossover.jsonl 2>> $OUT/err.log
done
cat $OUT/kprobe.jsonl $OUT/dyn.txt
python - <<'PY'
import json
for l in open("gpurun_out/scan/crossover.jsonl"):
    d = json.loads(l)
    print(d["lib"], d["model"], d["M"], d["kernel"], "%.3e" % d["firings_per_s"])
PY
