OUT=gpurun_out/r02v
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); print('warm')" > $OUT/warm.log 2>&1
python tools/c3_step_probe.py > $OUT/c3_step.txt 2>&1
python tools/resume_study.py C3 C2 C4 C5 > $OUT/next1_study.jsonl 2> $OUT/next1.err
python tools/lv_family.py --out $OUT/lv_family.jsonl > $OUT/lv_family.log 2>&1
