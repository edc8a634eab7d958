#!/bin/bash
# The GPU test suite on the bounds-checking library (libtetmf_b200_debug.so, -DTMF_DEBUG_CHECKS):
# every gathered / scattered index, cell, face position and block-local index the kernels derive
# is range-checked on the device and any violation fails the apply (see common.cuh).  This is
# the memcheck substitute: compute-sanitizer is closed on this GPU pool.  Log -> gpurun_out/.
set -u
mkdir -p gpurun_out
python -c "import os; os.environ['TMF_LIB']='debug'; import sys; sys.path.insert(0,'.'); from paper_2509_10226_b200 import _lib; print(_lib.lib().tmf_version().decode())" \
  > gpurun_out/debug_checks.log 2>&1
TMF_LIB=debug timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf >> gpurun_out/debug_checks.log 2>&1
echo "rc=$?" >> gpurun_out/debug_checks.log
tail -5 gpurun_out/debug_checks.log
