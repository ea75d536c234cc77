#!/bin/bash
# Round profile capture (run on the GPU box through gpurun, one GPU):
#   launch lists (cold-cache, serialised per-launch durations) for the three
#   measured workloads, and one `ncu --set full` capture of every kernel of
#   one solve, summarised to JSON by tools/ncu_summary.py.  Full reports stay
#   in /tmp on the box (they exceed gpurun's 64 MiB copy-back limit);
#   REPORTS=keep copies the general-path report back as well.
set -x
mkdir -p gpurun_out
B="python bench.py --no-cpu --no-e2e"
NM="ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv"
$NM --log-file gpurun_out/launches_noniter_cfg2.csv $B --steps 3 --warmup 2 > /tmp/l1.log 2>&1
$NM --log-file gpurun_out/launches_iter_cfg2.csv $B --solver iterative --steps 3 --warmup 2 > /tmp/l2.log 2>&1
$NM --log-file gpurun_out/launches_general_cfg4.csv $B --config cfg4 --steps 3 --warmup 2 > /tmp/l3.log 2>&1
NF="ncu -f --set full --clock-control none --import-source on -k regex:^k_"
$NF -c 12 -o /tmp/full_noniter_cfg2 $B --steps 1 --warmup 0 > /tmp/f1.log 2>&1
$NF -c 40 -o /tmp/full_iter_cfg2 $B --solver iterative --steps 1 --warmup 0 > /tmp/f2.log 2>&1
$NF -c 12 -o /tmp/full_general_cfg4 $B --config cfg4 --steps 1 --warmup 0 > /tmp/f3.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_full_noniter_cfg2.json /tmp/full_noniter_cfg2.ncu-rep
python tools/ncu_summary.py gpurun_out/ncu_full_iter_cfg2.json /tmp/full_iter_cfg2.ncu-rep
python tools/ncu_summary.py gpurun_out/ncu_full_general_cfg4.json /tmp/full_general_cfg4.ncu-rep
if [ "$REPORTS" = keep ]; then cp /tmp/full_general_cfg4.ncu-rep gpurun_out/; fi
ls -la gpurun_out /tmp/*.ncu-rep
