#!/bin/bash
# The GPU suite under the device-assert build (-DDDKS_DEBUG: DDKS_ASSERT bounds checks in every kernel), then a larger
# seeded fuzz of the rank-lane count on the same build. Run on a scratch copy of the library; the shipped .so is rebuilt after.
O=gpurun_out; mkdir -p $O
DDKS_DEBUG=1 python -c "from paper_2106_13706_b200 import build; build.build(force=True)" > $O/r2f_debug_build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > $O/r2f_debug_asserts_gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/r2f_debug_asserts_gpu_tests.log
DDKS_FUZZ_CASES=600 timeout 900 python -m pytest tests/test_rank_gpu.py -m gpu -q -k fuzz > $O/r2f_rank_fuzz_200_debug.log 2>&1; echo "pytest rc=$?" >> $O/r2f_rank_fuzz_200_debug.log
tail -3 $O/r2f_debug_asserts_gpu_tests.log; tail -3 $O/r2f_rank_fuzz_200_debug.log
