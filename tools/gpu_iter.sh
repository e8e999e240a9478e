#!/bin/bash
# Development iteration on one B200: slab / guard / Krylov tests, a short bench (formal solvers,
# Krylov), and an ncu capture of the cfg5 tile and source-plane kernels.
O=gpurun_out
T=/tmp/ncu_iter
mkdir -p $O $T
python -m pytest tests/test_gpu_slab.py tests/test_gpu_guards.py tests/test_gpu_krylov.py -x -q 2>&1 | tail -5
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-lattice --no-reference-as-shipped > $O/bench_iter.jsonl 2> $O/bench_iter.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_iter.jsonl").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"])
print("formal", json.dumps(d.get("formal_solvers_cfg2"), indent=0))
print("krylov", json.dumps(d.get("krylov_cfg2")))
PY
[ "${1:-5}" = "skip" ] && exit 0
NCU="ncu --set full --clock-control none --import-source on"
for cfg in ${1:-5}; do
$NCU -k regex:'lattice_mom_tile' --launch-skip 40 -c 1 -f -o $T/tile$cfg python tools/prof_lattice.py $cfg > $O/ncu_tile.log 2>&1
python tools/ncu_summary.py $T/tile$cfg.ncu-rep $O/iter_ncu_tile_cfg$cfg.txt > /dev/null 2>&1
python tools/ncu_stalls.py $T/tile$cfg.ncu-rep 30 4 >> $O/iter_ncu_tile_cfg$cfg.txt 2>&1
$NCU -k regex:'lattice_splane_pm' --launch-skip 40 -c 1 -f -o $T/spl$cfg python tools/prof_lattice.py $cfg > $O/ncu_spl.log 2>&1
python tools/ncu_summary.py $T/spl$cfg.ncu-rep $O/iter_ncu_splane_cfg$cfg.txt > /dev/null 2>&1
done
