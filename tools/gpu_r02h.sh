OUT=gpurun_out/r02h
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -v -x --timeout 60 -k "warp" > $OUT/pytest_warp.log 2>&1; echo pytest=$?
