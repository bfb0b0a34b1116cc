#!/bin/bash
# averaged reconstruction: warp-level MMA (default for 16 <= W r <= 64) vs the earlier kernels
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_recon.py tests/test_gpu_engine.py -x -q -p no:cacheprovider > gpurun_out/rm_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/rm_pytest.log
rm -f gpurun_out/rm.txt
for r in 4 8 16; do
  echo "mma r$r $(timeout 300 python tools/recon_probe.py --rank $r --worlds 1,2,4,8 2>&1 | tail -1)" >> gpurun_out/rm.txt
  echo "old r$r $(EDGC_RECON_MMA_MIN=1000 timeout 300 python tools/recon_probe.py --rank $r --worlds 1,2,4,8 2>&1 | tail -1)" >> gpurun_out/rm.txt
done
exit 0
