#!/bin/bash
# Compile-time variants of a kernel file, built and timed on the GPU box (development
# experiment; the tree's own library is restored at the end).
#   OBJ=lattice|sigma_fused|...  CMD="python tools/time_lattice.py 4 5"  KPAT=<ptxas log pattern>
#   bash tools/gpu_variants.sh "-DFOO=1" "-DFOO=2" ...
OBJ=${OBJ:-lattice}
CMD=${CMD:-python tools/time_lattice.py 4 5}
cp paper_2602_21958_b200/librtk_b200.so /tmp/librtk_keep.so
for v in "$@"; do
  echo "== variant $v"
  rm -f build/rtk/$OBJ.o
  make -C paper_2602_21958_b200/csrc -j8 NVCC="/usr/local/cuda/bin/nvcc $v" > /tmp/build_variant.log 2>&1 || { tail -5 /tmp/build_variant.log; continue; }
  [ -n "${KPAT:-}" ] && grep -A2 "$KPAT" build/rtk/$OBJ.o.ptxas.log | grep -E "spill|registers"
  $CMD 2>&1 | tail -${NTAIL:-2}
  [ -n "${CMD2:-}" ] && $CMD2 2>&1 | tail -${NTAIL2:-3}
done
cp /tmp/librtk_keep.so paper_2602_21958_b200/librtk_b200.so
rm -f build/rtk/$OBJ.o
