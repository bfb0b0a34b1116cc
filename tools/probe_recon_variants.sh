mkdir -p gpurun_out; rm -f gpurun_out/rv.txt
for v in base m16_3 m16_4 m32_1 m32_3r4; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  echo "$v $(timeout 300 python tools/recon_probe.py --rank 4 --worlds 4,8 2>&1 | tail -1)" >> gpurun_out/rv.txt
done
exit 0
