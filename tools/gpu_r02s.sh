OUT=gpurun_out/r02s
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); print('warm')" > $OUT/warm.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "thread or ws2" > $OUT/pytest_thread.log 2>&1; echo pytest=$?
for k in ws ws2 single thread2; do
  python tools/kprobe.py --config C2 --t-end 2 --kernel $k >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C1 --kernel $k >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C2 --t-end 2 --replicas 64 --kernel $k >> $OUT/probe.jsonl 2>>$OUT/err.log
done
python tools/kprobe.py --config C3 --kernel single >> $OUT/probe.jsonl 2>>$OUT/err.log
python tools/kprobe.py --config C3 --kernel thread2 >> $OUT/probe.jsonl 2>>$OUT/err.log
