OUT=gpurun_out/r02m
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); print('warm')" > $OUT/warm.log 2>&1
for v in "777 default" "700 default" "650 default"; do
  timeout 45 python tools/dbg_cases2.py $v >> $OUT/cases2.log 2>&1; echo "$v rc=$?" >> $OUT/cases2.log
done
