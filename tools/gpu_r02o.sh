OUT=gpurun_out/r02o
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); print('warm')" > $OUT/warm.log 2>&1
CWC_PARITY_FULL=1 CWC_PARITY_OUT=$OUT/parity timeout 2700 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_parity_full.py -v -p no:cacheprovider --durations=12 > $OUT/pytest_parity.log 2>&1; echo pytest=$?
