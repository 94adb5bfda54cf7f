OUT=gpurun_out/r02u
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); print('warm')" > $OUT/warm.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_resume.py -q -x -k "warp or shard or modes or overflow or stall" > $OUT/pytest_warp.log 2>&1; echo pytest=$?
python tools/kprobe.py --config C4 >> $OUT/probe.jsonl 2>>$OUT/err.log
python tools/kprobe.py --config C5 >> $OUT/probe.jsonl 2>>$OUT/err.log
