OUT=gpurun_out/r02t
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); print('warm')" > $OUT/warm.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ws2" > $OUT/pytest_ws2.log 2>&1; echo pytest=$?
for lib in libcwcsim libcwcsim_ws2p1; do
  L=paper_1010_2438_b200/$lib.so
  python tools/kprobe.py --config C2 --t-end 2 --kernel ws2 --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C2 --t-end 2 --replicas 64 --kernel ws2 --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C1 --kernel ws2 --lib $L >> $OUT/probe.jsonl 2>>$OUT/err.log
done
python tools/kprobe.py --config C2 --t-end 2 --kernel single >> $OUT/probe.jsonl 2>>$OUT/err.log
