#!/bin/bash
# instrumented copy of the library (prof/liblyapir_prof$1.so): gje_ip.cu with -DLYAP_PANEL_PROF [-DLYAP_IP_ABLATE=$1], the other objects as built
set -e
cd "$(dirname "$0")/../paper_2510_02126_b200"
python build.py > /dev/null
mkdir -p prof
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
EXTRA=""; [ -n "$1" ] && EXTRA="-DLYAP_IP_ABLATE=$1"
nvcc $FL -DLYAP_PANEL_PROF $EXTRA -c csrc/gje_ip.cu -o prof/gje_ip$1.o
OBJS=$(ls build/*.o | grep -v gje_ip.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o prof/liblyapir_prof$1.so $OBJS prof/gje_ip$1.o
echo prof/liblyapir_prof$1.so
