#!/bin/bash
# DMMA (FP64 tensor) sub-pipe utilisation of the fused Sigma kernel and of the unfused DMMA GEMM at
# cfg2 -> gpurun_out/r02_ncu_dmma_pipes.txt (the format bench.py's ncu_dmma_pipes() reads).
O=gpurun_out/r02_ncu_dmma_pipes.txt
M=gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
mkdir -p gpurun_out
echo "# DMMA (FP64 tensor) pipe utilisation from ncu (cfg2, one launch each; round 2 final tree)" > $O
ncu --metrics $M --clock-control none -k regex:sigma_fused --launch-skip 3 -c 1 --csv --log-file /tmp/dm_f.csv python tools/prof_cfg2.py ie 5 > /dev/null 2>&1
RTK_SIGMA_UNFUSED=1 ncu --metrics $M --clock-control none -k regex:redistribute_dmma --launch-skip 3 -c 1 --csv --log-file /tmp/dm_u.csv python tools/prof_cfg2.py ie 5 > /dev/null 2>&1
python - <<'PY' >> $O
import csv
for path in ("/tmp/dm_u.csv", "/tmp/dm_f.csv"):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    if not rows:
        continue
    name = rows[0][4]
    print("== " + name[:100])
    print("  raw: " + ", ".join(f"{r[-3]}={r[-1]}{r[-2]}" for r in rows))
PY
cat $O | cut -c1-400
