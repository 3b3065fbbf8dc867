#!/bin/bash
# quick GPU check: selected GPU tests (-k expr or all), then the bench A/B specs
# usage: bash tools/gpu_quick2.sh OUTNAME "pytest -k expr or ''" "label|ENV|lib" ...
O=gpurun_out/$1; K=$2; shift 2; mkdir -p $O
if [ -n "$K" ]; then
  if [ "$K" = "all" ]; then timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.txt 2>&1
  else timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K" > $O/tests.txt 2>&1; fi
  tail -15 $O/tests.txt
fi
[ $# -gt 0 ] && bash tools/gpu_ab2.sh $O "$@"
