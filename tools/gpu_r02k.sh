OUT=gpurun_out/r02k
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); print('warm')" > $OUT/warm.log 2>&1
timeout 60 python tools/dbg_cases.py c1 >> $OUT/cases.log 2>&1; echo c1=$? >> $OUT/cases.log
timeout 60 python tools/dbg_cases.py decay paper_1010_2438_b200/libcwcsim_oldwarp.so >> $OUT/cases.log 2>&1; echo decay_old=$? >> $OUT/cases.log
timeout 60 python tools/dbg_cases.py decay >> $OUT/cases.log 2>&1; echo decay=$? >> $OUT/cases.log
