set -x
timeout 300 python tools/pass1_ab.py --rank 128 --iters 3
EDGC_LIB_PATH=alt_libs/efnoload.so timeout 300 python tools/pass1_ab.py --rank 128 --iters 3
EDGC_LIB_PATH=alt_libs/efnostore.so timeout 300 python tools/pass1_ab.py --rank 128 --iters 3
