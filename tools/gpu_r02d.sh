OUT=gpurun_out/r02d
mkdir -p $OUT
./tools/pipebench/pipe_bench > $OUT/pipe_bench.json 2>&1; echo pipe=$?
for lib in libcwcsim libcwcsim_nowide; do
  PROBE_LIB=paper_1010_2438_b200/$lib.so PROBE_R=32,4736,9472,16384 python tools/c2_probe.py 2.0 > $OUT/probe_$lib.jsonl 2>&1; echo $lib=$?
done
for R in 32 4736 16384; do python tools/ws_prof.py --config C2 --t-end 2 --replicas $R --lib paper_1010_2438_b200/libcwcsim_wsprof.so >> $OUT/wsprof.txt 2>&1; done
