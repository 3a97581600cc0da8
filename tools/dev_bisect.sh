mkdir -p gpurun_out
FBP_NVCC_FLAGS=-DFBP_DEV_MASK=1 python -m paper_2007_06289_b200.build > gpurun_out/devbuild.log 2>&1 || { echo BUILD_FAIL; tail gpurun_out/devbuild.log; }
for m in 0 16 8 24; do for mode in bp rec; do FBP_DBG=$m timeout 60 python tools/dev_bisect.py 512 $mode 2>&1 | grep DBG; done; done
