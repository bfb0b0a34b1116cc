#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_compress.py tests/test_gpu_engine.py tests/test_calibrate.py -x -q -p no:cacheprovider > gpurun_out/zb_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/zb_pytest.log
timeout 300 python tools/api_probe.py > gpurun_out/zb_api.log 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/zb_bench100_$i.log 2>&1; done
exit 0
