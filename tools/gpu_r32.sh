set -x
timeout 300 python tools/recon_probe.py --worlds 4,8
EDGC_LIB_PATH=alt_libs/r32b1.so timeout 300 python tools/recon_probe.py --worlds 4,8
