OUT=gpurun_out/r02q
mkdir -p $OUT
for R in 16384 18944 37888 75776; do
  python tools/kprobe.py --config C2 --t-end 1 --replicas $R --kernel single >> $OUT/probe.jsonl 2>>$OUT/err.log
  python tools/kprobe.py --config C2 --t-end 1 --replicas $R --kernel ws >> $OUT/probe.jsonl 2>>$OUT/err.log
done
for R in 16 32 64; do python tools/kprobe.py --config C3 --replicas $R --kernel single >> $OUT/probe.jsonl 2>>$OUT/err.log; done
python - > $OUT/memset.txt 2>&1 <<'PY'
import torch
x = torch.empty(53 * 2**20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); x.zero_(); e1.record(); torch.cuda.synchronize()
    import ctypes
    print("torch zero_ 53MB ms", e0.elapsed_time(e1))
cudart = ctypes.CDLL("libcudart.so.12") if False else None
PY
python tools/c3_step_probe.py > $OUT/c3_step.txt 2>&1
