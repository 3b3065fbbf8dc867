#!/bin/bash
# build an A/B variant of the library: tools/build_variant.sh NAME "-DFLAG=.. ..." -> paper_2112_07075_b200/lib_NAME.so
cd /root/repo || exit 1
N=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared $* \
  -Xptxas -v -o paper_2112_07075_b200/lib_$N.so paper_2112_07075_b200/csrc/hx_api.cu > /tmp/ptxas_$N.log 2>&1 || { tail /tmp/ptxas_$N.log; exit 1; }
grep -A1 "k_mass_brickILi3ELi3E" /tmp/ptxas_$N.log | grep -E "registers|spill" | head -3
echo "built lib_$N.so"
