#!/bin/bash
# Round-end evidence on one B200: full GPU test suite, smoke, both bench arms, the ncu launch
# list of the bench step and --set full summaries of the dominant kernels.
O=gpurun_out
T=/tmp/ncu_round
mkdir -p $O $T
nvidia-smi -L > $O/gpu.txt
python -m pytest tests -m gpu -x -q > $O/r02_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/r02_smoke.log 2>&1; tail -1 $O/r02_smoke.log
python bench.py --impl reference > $O/r02_bench_cfg2_reference.jsonl 2> $O/bench_ref.err; echo "ref rc=$?"
python bench.py > $O/r02_bench_cfg2.jsonl 2> $O/bench.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/r02_launches_cfg2_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gmres --no-lattice --no-reference-as-shipped > $O/ncu_bench.log 2>&1; echo "launch list rc=$?"
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:'sweep1d_tma|sigma_fused' --launch-skip 4 -c 2 -f -o $T/cfg2 python tools/prof_cfg2.py ie 4 > $O/ncu_cfg2.log 2>&1
python tools/ncu_summary.py $T/cfg2.ncu-rep $O/r02_ncu_cfg2_kernels.txt > /dev/null 2>&1
$NCU -k regex:'sweep1d_tma' --launch-skip 2 -c 1 -f -o $T/cfg2_ep python tools/prof_cfg2.py exp_parabolic 4 > $O/ncu_cfg2_ep.log 2>&1
python tools/ncu_summary.py $T/cfg2_ep.ncu-rep $O/r02_ncu_sweep_exp_parabolic.txt > /dev/null 2>&1
$NCU -k regex:'sweep1d_tma' --launch-skip 2 -c 1 -f -o $T/cfg2_el python tools/prof_cfg2.py exp_linear 4 > $O/ncu_cfg2_el.log 2>&1
python tools/ncu_summary.py $T/cfg2_el.ncu-rep $O/r02_ncu_sweep_exp_linear.txt > /dev/null 2>&1
for cfg in 4 5 3; do
  skip=40; [ $cfg = 3 ] && skip=0
  $NCU -k regex:'lattice_mom_tile|lattice_int_smem' --launch-skip $skip -c 1 -f -o $T/lattice_cfg$cfg python tools/prof_lattice.py $cfg > $O/ncu_lattice_$cfg.log 2>&1
  python tools/ncu_summary.py $T/lattice_cfg$cfg.ncu-rep $O/r02_ncu_lattice_cfg$cfg.txt > /dev/null 2>&1
  python tools/ncu_stalls.py $T/lattice_cfg$cfg.ncu-rep 12 2 >> $O/r02_ncu_lattice_cfg$cfg.txt 2>&1
  $NCU -k regex:'lattice_splane|expand_nodes|lattice_mom_reduce|redistribute' --launch-skip $skip -c 3 -f -o $T/lattice_aux_cfg$cfg python tools/prof_lattice.py $cfg > $O/ncu_lattice_aux_$cfg.log 2>&1
  python tools/ncu_summary.py $T/lattice_aux_cfg$cfg.ncu-rep $O/r02_ncu_lattice_aux_cfg$cfg.txt > /dev/null 2>&1
done
$NCU -k regex:'scale_kernel' --launch-skip 6 -c 1 -f -o $T/scale python tools/prof_krylov.py cgs2 8 > $O/ncu_scale.log 2>&1
python tools/ncu_summary.py $T/scale.ncu-rep $O/r02_ncu_krylov_scale.txt > /dev/null 2>&1
du -sh $O
