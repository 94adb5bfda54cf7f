#!/bin/bash
# Build an experiment variant of libcwcsim.so: tools/build_variant.sh TAG "NVCC FLAGS"
# -> paper_1010_2438_b200/libcwcsim_TAG.so (run it with tools/variant_run.py)
CWC_BUILD_TAG=$1 NVCC_EXTRA="$2" python -c "from paper_1010_2438_b200 import _build; print(_build.build())"
