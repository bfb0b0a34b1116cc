#!/bin/bash
# averaged reconstruction on CUDA cores vs forced onto the tensor cores (EDGC_TC_RECON_MIN=8)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_recon.py -x -q -p no:cacheprovider > gpurun_out/tcr_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/tcr_pytest.log
echo "cuda $(timeout 300 python tools/recon_probe.py --rank 4 --worlds 1,2,4,8 2>&1 | tail -1)" > gpurun_out/tcr.txt
echo "tc $(EDGC_TC_RECON_MIN=8 timeout 300 python tools/recon_probe.py --rank 4 --worlds 2,4,8 2>&1 | tail -1)" >> gpurun_out/tcr.txt
echo "cuda8 $(timeout 300 python tools/recon_probe.py --rank 8 --worlds 1,2,4,8 2>&1 | tail -1)" >> gpurun_out/tcr.txt
echo "tc8 $(EDGC_TC_RECON_MIN=8 timeout 300 python tools/recon_probe.py --rank 8 --worlds 1,2,4,8 2>&1 | tail -1)" >> gpurun_out/tcr.txt
exit 0
