OUT=gpurun_out/r02r
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); print('warm')" > $OUT/warm.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "thread" > $OUT/pytest_thread.log 2>&1; echo pytest=$?
for k in single thread2; do
  python tools/kprobe.py --config C2 --t-end 2 --kernel $k >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C3 --kernel $k >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C2 --t-end 2 --replicas 32 --kernel $k >> $OUT/probe.jsonl 2>>$OUT/err.log
done
