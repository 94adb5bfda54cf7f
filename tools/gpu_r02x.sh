# A/B against the committed build (libcwcsim.so): dependency-entry prefetch (pref), + division overlapped with the
# selection's first stage (pref2), + next draw broadcast ahead of the re-sum (pref3) in the one-per-warp kernel;
# pref4 = pref3 + the division overlap in the two-per-warp kernel
OUT=gpurun_out/pref
mkdir -p $OUT
for rep in 1 2; do
for lib in libcwcsim.so libcwcsim_pref2.so libcwcsim_pref3.so libcwcsim_pref4.so; do
  python tools/kprobe.py --config C5 --lib paper_1010_2438_b200/$lib >> $OUT/kprobe.jsonl 2>> $OUT/err.log
  python tools/kprobe.py --config C4 --kernel warp --t-end 0.3 --lib paper_1010_2438_b200/$lib >> $OUT/kprobe.jsonl 2>> $OUT/err.log
done
for lib in libcwcsim.so libcwcsim_pref4.so; do
  python tools/kprobe.py --config C4 --lib paper_1010_2438_b200/$lib >> $OUT/kprobe.jsonl 2>> $OUT/err.log
done
done
python - <<'PY'
import json
for l in open("gpurun_out/pref/kprobe.jsonl"):
    d = json.loads(l)
    print(d["tag"], d["config"], d["kernel"], "%.4e" % d["firings_per_s"], "%.2f ms" % d["kernel_ms"])
PY
