OUT=gpurun_out/r02j
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); print('warm')" > $OUT/warm.log 2>&1
for c in decay stall dimer c3one c3short c3sweep; do timeout 60 python tools/dbg_cases.py $c >> $OUT/cases.log 2>&1; echo $c=$? >> $OUT/cases.log; done
