#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_recon.py -x -q -p no:cacheprovider > gpurun_out/x_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/x_pytest.log
for t in 1000 8 16 32; do
EDGC_TC_RECON_MIN=$t timeout 300 python tools/recon_probe.py --rank 4 > gpurun_out/x_recon_r4_min$t.log 2>&1
done
EDGC_TC_RECON_MIN=1000 timeout 300 python tools/recon_probe.py --rank 8 > gpurun_out/x_recon_r8_cc.log 2>&1
timeout 300 python tools/recon_probe.py --rank 8 > gpurun_out/x_recon_r8_tc.log 2>&1
exit 0
