# Developer: dev build, FBP_VERBOSE launch geometry + KS/KB times under skip masks
FBP_NVCC_FLAGS=-DFBP_DEV_MASK=1 python -m paper_2007_06289_b200.build > /dev/null 2>&1 || echo BUILD_FAIL
FBP_VERBOSE=1 timeout 120 python tools/dev_timing2.py ${N:-2048} ${B:-16} 2>&1 | grep -m1 "sweep:"
for m in ${MASKS:-0 8 32 64}; do FBP_DBG=$m timeout 120 python tools/dev_timing2.py ${N:-2048} ${B:-16} 2>&1 | grep DBG; done
