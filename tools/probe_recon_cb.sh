#!/bin/bash
# W r = 32 reconstruction: 512-column blocks per tile (one P tile load for all) A/B
mkdir -p gpurun_out/rcb; O=gpurun_out/rcb; rm -f $O/ab.txt
timeout 300 python -m pytest tests/test_gpu_recon.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for lib in default alt_libs/cb2.so alt_libs/cb4.so alt_libs/cb8.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  echo "$lib r4 $(timeout 300 python tools/recon_probe.py --rank 4 --worlds 1,8 2>/dev/null | tail -1)" >> $O/ab.txt
  echo "$lib r32 $(timeout 300 python tools/recon_probe.py --rank 32 --worlds 1 2>/dev/null | tail -1)" >> $O/ab.txt
  echo "$lib r8 $(timeout 300 python tools/recon_probe.py --rank 8 --worlds 4 2>/dev/null | tail -1)" >> $O/ab.txt
done
exit 0
