# compute-sanitizer memcheck (one tool per call) on small runs of every kernel variant.
set -x
OUT=gpurun_out/${TAG:-sanitize}
mkdir -p $OUT
run() { name=$1; shift; "$@" > $OUT/plain_$name.log 2>&1 && \
  compute-sanitizer --tool ${TOOL:-memcheck} --error-exitcode 9 "$@" > $OUT/${TOOL:-memcheck}_$name.log 2>&1; echo $name=$?; }
run c2_ws python tools/run_case.py --config C2 --t-end 0.05 --replicas 256
run c3_ws python tools/run_case.py --config C3 --t-end 5.0 --replicas 4
run c2_thread1 python tools/run_case.py --config C2 --t-end 0.05 --replicas 256 --block-threads 64
run c4_warp2 python tools/run_case.py --config C4 --t-end 0.02 --replicas 64
run c5_warp python tools/run_case.py --config C5 --t-end 0.05 --replicas 64
tail -n 3 $OUT/${TOOL:-memcheck}_*.log
