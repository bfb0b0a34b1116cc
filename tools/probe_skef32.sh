#!/bin/bash
# rank 32: tcgen05 TcEF + TcPraw (default) vs the fused CUDA-core EF + P_raw (alt_libs/s32*.so)
mkdir -p gpurun_out/s32; O=gpurun_out/s32; rm -f $O/ab.txt
EDGC_LIB_PATH=$PWD/alt_libs/s32a.so timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compress.py tests/test_gpu_dp.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for lib in default alt_libs/s32a.so alt_libs/s32b.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  for r in 24 32; do
  echo "$lib $r $(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> $O/ab.txt
  done
done
exit 0
