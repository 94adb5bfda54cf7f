# A/B of the nearly-full-chunk re-sum (libcwcsim_chunk.so) against the committed build: C5, C4 (warp kernel forced), LV-129
OUT=gpurun_out/chunk
mkdir -p $OUT
for rep in 1 2; do
for lib in libcwcsim.so libcwcsim_chunk.so; do
  python tools/kprobe.py --config C5 --lib paper_1010_2438_b200/$lib >> $OUT/kprobe.jsonl 2>> $OUT/err.log
  python tools/kprobe.py --config C4 --kernel warp --t-end 0.3 --lib paper_1010_2438_b200/$lib >> $OUT/kprobe.jsonl 2>> $OUT/err.log
done
done
cat $OUT/kprobe.jsonl
