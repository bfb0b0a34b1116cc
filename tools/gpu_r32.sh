set -x
timeout 300 python tools/recon_probe.py --worlds 1,8
EDGC_LIB_PATH=alt_libs/r32r4.so timeout 300 python tools/recon_probe.py --worlds 1,8
