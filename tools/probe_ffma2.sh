#!/bin/bash
# FFMA2 A/B: skinny GEMM / EF tiles (ranks 8 / 16 / 32) and the reconstruction's W r threshold
mkdir -p gpurun_out/f2ab; O=gpurun_out/f2ab; rm -f $O/ab.txt
timeout 600 python -m pytest tests/test_gpu_recon.py tests/test_gpu_engine.py tests/test_gpu_compress.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for lib in default alt_libs/noskf2.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  for r in 8 16 32; do
    echo "$lib $r $(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> $O/ab.txt
  done
done
for lib in default alt_libs/f2all.so alt_libs/f2only32.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  echo "$lib recon_r4 $(timeout 300 python tools/recon_probe.py --rank 4 2>/dev/null | tail -1)" >> $O/recon.txt
  echo "$lib recon_r8 $(timeout 300 python tools/recon_probe.py --rank 8 --worlds 1,2 2>/dev/null | tail -1)" >> $O/recon.txt
done
exit 0
