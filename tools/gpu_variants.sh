#!/bin/bash
# Compile-time variants of the tiled moment kernel, built and timed on the GPU box
# (development experiment; the tree's own library is restored at the end).
cp paper_2602_21958_b200/librtk_b200.so /tmp/librtk_keep.so
for v in "$@"; do
  echo "== variant $v"
  rm -f build/rtk/lattice.o
  make -C paper_2602_21958_b200/csrc -j8 NVCC="/usr/local/cuda/bin/nvcc $v" > /tmp/build_variant.log 2>&1 || { tail -5 /tmp/build_variant.log; continue; }
  grep -A2 "${KPAT:-lattice_mom_tile_kernelILi0ELi6ELi16ELi16E}" build/rtk/lattice.o.ptxas.log | grep -E "spill|registers"
  python tools/time_lattice.py ${CFGS:-4 5} 2>&1 | tail -${NTAIL:-2}
done
cp /tmp/librtk_keep.so paper_2602_21958_b200/librtk_b200.so
