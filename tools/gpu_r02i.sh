OUT=gpurun_out/r02i
mkdir -p $OUT
timeout 120 python tools/dbg_c3warp.py paper_1010_2438_b200/libcwcsim_dbg.so > $OUT/dbg.log 2>&1; echo dbg=$?
