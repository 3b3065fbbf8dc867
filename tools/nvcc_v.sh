#!/bin/bash
# build the in-tree library with ptxas resource usage (-Xptxas -v) into /tmp/ptxas.log;
# prints errors and the register / spill lines of kernels matching $1
cd /root/repo || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared -Xptxas -v \
  -o paper_2112_07075_b200/libb200hydro.so.tmp paper_2112_07075_b200/csrc/hx_api.cu > /tmp/ptxas.log 2>&1
rc=$?
grep -E "error" /tmp/ptxas.log | head -20
[ $rc -eq 0 ] && mv paper_2112_07075_b200/libb200hydro.so.tmp paper_2112_07075_b200/libb200hydro.so && echo "BUILD OK"
python3 tools/ptxas_regs.py /tmp/ptxas.log ${@:-k_rates_pc}
