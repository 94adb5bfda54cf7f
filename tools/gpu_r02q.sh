OUT=gpurun_out/r02q
mkdir -p $OUT
for R in 16384 18944 37888 75776; do
  python tools/kprobe.py --config C2 --t-end 1 --replicas $R --kernel single >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C2 --t-end 1 --replicas $R --kernel ws >> $OUT/probe.jsonl 2>>$OUT/err.log
done
for R in 16 32 64; do python tools/kprobe.py --config C3 --replicas $R --kernel single >> $OUT/probe.jsonl 2>>$OUT/err.log; done
