#!/bin/bash
# W r = 32 reconstruction: FFMA vs FFMA2 (paired columns) A/B
mkdir -p gpurun_out/rf2; O=gpurun_out/rf2; rm -f $O/ab.txt
EDGC_LIB_PATH=$PWD/alt_libs/ffma2.so timeout 300 python -m pytest tests/test_gpu_recon.py tests/test_gpu_engine.py -x -q -p no:cacheprovider -k "recon or rank or chained" > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do
for lib in default alt_libs/ffma2.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  echo "$lib r4 $(timeout 300 python tools/recon_probe.py --rank 4 --worlds 8 2>/dev/null | tail -1)" >> $O/ab.txt
  echo "$lib r32 $(timeout 300 python tools/recon_probe.py --rank 32 --worlds 1 2>/dev/null | tail -1)" >> $O/ab.txt
done
done
exit 0
