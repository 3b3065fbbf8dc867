#!/bin/bash
# build the library in-tree and fail loudly
cd /root/repo || exit 1
python -m paper_2112_07075_b200.build 2>&1 | grep -iE "error|warning" | grep -v Remark
test paper_2112_07075_b200/libb200hydro.so -nt paper_2112_07075_b200/csrc/hx_kernels.cuh && test paper_2112_07075_b200/libb200hydro.so -nt paper_2112_07075_b200/csrc/hx_api.cu && echo "BUILD OK" || { echo "BUILD FAILED"; exit 1; }
