#!/bin/bash
# Round evidence on one B200: ncu --set full captures of the Krylov and lattice kernels and
# compute-sanitizer passes over every mbarrier / TMA / cluster kernel family.  Text summaries
# go to gpurun_out/ (the .ncu-rep files stay in /tmp except the small ones: 64 MiB return limit).
set -u
O=gpurun_out
T=/tmp/ncu_r02
mkdir -p $O $T
NCU="ncu --set full --clock-control none --import-source on"
summ() {  # summ <rep> <out.txt>: details summary + the 25 hottest source lines by stall samples
  python tools/ncu_summary.py $1 $2 > /dev/null 2>&1
  python tools/ncu_stalls.py $1 >> $2 2>&1
}
what=${1:-all}
if [ $what = all ] || [ $what = krylov ]; then
python tools/prof_krylov.py cgs2 8 > $O/prof_krylov_plain.log 2>&1 || exit 1
$NCU -k regex:'cgs_pass|scale_kernel' --launch-skip 24 -c 4 -f -o $T/krylov_cgs2 python tools/prof_krylov.py cgs2 8 > $O/ncu_krylov_cgs2.log 2>&1
summ $T/krylov_cgs2.ncu-rep $O/r02_ncu_krylov_cgs2.txt
$NCU -k regex:'mgs_pass' --launch-skip 40 -c 2 -f -o $T/krylov_mgs python tools/prof_krylov.py mgs 8 > $O/ncu_krylov_mgs.log 2>&1
summ $T/krylov_mgs.ncu-rep $O/r02_ncu_krylov_mgs.txt
fi
if [ $what = all ] || [ $what = lattice ]; then
for cfg in 4 5 3; do
  python tools/prof_lattice.py $cfg > $O/prof_lattice_$cfg.log 2>&1 || continue
  skip=40; [ $cfg = 3 ] && skip=0
  $NCU -k regex:'lattice_mom_tile|lattice_int_smem|lattice_mom_group' --launch-skip $skip -c 1 -f -o $T/lattice_cfg$cfg python tools/prof_lattice.py $cfg > $O/ncu_lattice_$cfg.log 2>&1
  summ $T/lattice_cfg$cfg.ncu-rep $O/r02_ncu_lattice_cfg$cfg.txt
  [ $(stat -c %s $T/lattice_cfg$cfg.ncu-rep) -lt 15000000 ] && cp $T/lattice_cfg$cfg.ncu-rep $O/
  $NCU -k regex:'lattice_splane|expand_nodes|expand_kernel|lattice_mom_reduce|redistribute' --launch-skip $skip -c 3 -f -o $T/lattice_aux_cfg$cfg python tools/prof_lattice.py $cfg > $O/ncu_lattice_aux_$cfg.log 2>&1
  python tools/ncu_summary.py $T/lattice_aux_cfg$cfg.ncu-rep $O/r02_ncu_lattice_aux_cfg$cfg.txt > /dev/null 2>&1
done
fi
if [ $what = all ] || [ $what = sanitizer ]; then
rm -f $O/r02_sanitizer_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 7 python tools/sanitize_driver.py > $O/r02_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/r02_sanitizer_summary.txt
  tail -5 $O/r02_sanitizer_$tool.log
done
cat $O/r02_sanitizer_summary.txt
fi
du -sh $O
