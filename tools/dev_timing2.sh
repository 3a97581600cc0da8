FBP_NVCC_FLAGS=-DFBP_DEV_MASK=1 python -m paper_2007_06289_b200.build > /dev/null 2>&1 || echo BUILD_FAIL
for m in ${MASKS:-0 8 1 2 3 32 64 96 99 107}; do FBP_DBG=$m timeout 120 python tools/dev_timing2.py ${N:-2048} ${B:-16} 2>&1 | grep DBG; done
