OUT=gpurun_out/r02l
mkdir -p $OUT
NREP=777 timeout 120 python tools/dbg_monitor.py paper_1010_2438_b200/libcwcsim_dbg.so decay > $OUT/mon_decay.log 2>&1; echo decay=$?
NREP=200 timeout 120 python tools/dbg_monitor.py paper_1010_2438_b200/libcwcsim_dbg.so decay > $OUT/mon_decay200.log 2>&1; echo decay=$?
