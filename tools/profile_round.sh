#!/bin/bash
# Round profile capture (run on the GPU box through gpurun, one GPU):
#   launch lists (cold-cache, serialised per-launch durations) of the
#   default bench command and the main workloads, and `ncu --set full`
#   captures of one solve, summarised to JSON by tools/ncu_summary.py.  Full
#   reports stay in /tmp on the box (they exceed gpurun's 64 MiB copy-back).
#   $1 = round tag (r02).
T=${1:-r02}
set -x
mkdir -p gpurun_out/prof_$T
O=gpurun_out/prof_$T
B="python bench.py --no-cpu --no-e2e"
NM="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
# the default bench command itself (bench.py --steps 2 --warmup 1), every kernel
$NM --log-file $O/launches_bench_default.csv python bench.py --steps 2 --warmup 1 --no-cpu > /tmp/l0.log 2>&1
$NM -k regex:^k_ --log-file $O/launches_noniter_cfg2.csv $B --steps 3 --warmup 2 > /tmp/l1.log 2>&1
$NM -k regex:^k_ --log-file $O/launches_iter_cfg2.csv $B --solver iterative --steps 3 --warmup 2 > /tmp/l2.log 2>&1
$NM -k regex:^k_ --log-file $O/launches_general_cfg4.csv $B --config cfg4 --steps 3 --warmup 2 > /tmp/l3.log 2>&1
$NM -k regex:^k_ --log-file $O/launches_general_cfg5_k16384.csv $B --config cfg5 --cfg5-general --k 16384 --steps 1 --warmup 1 > /tmp/l4.log 2>&1
NF="ncu -f --set full --clock-control none --import-source on -k regex:^k_"
$NF -c 12 -o /tmp/full_noniter_cfg2 $B --steps 1 --warmup 0 > /tmp/f1.log 2>&1
$NF -c 40 -o /tmp/full_iter_cfg2 $B --solver iterative --steps 1 --warmup 0 > /tmp/f2.log 2>&1
$NF -c 14 -o /tmp/full_general_cfg4 $B --config cfg4 --steps 1 --warmup 0 > /tmp/f3.log 2>&1
$NF -c 24 -o /tmp/full_general_c5g16k $B --config cfg5 --cfg5-general --k 16384 --steps 1 --warmup 0 > /tmp/f4.log 2>&1
for r in noniter_cfg2 iter_cfg2 general_cfg4 general_c5g16k; do
  python tools/ncu_summary.py $O/ncu_full_$r.json /tmp/full_$r.ncu-rep
done
for f in $O/launches_*.csv; do echo "== $f"; python tools/launches.py $f 2; done > $O/launches_summary.txt
ls -la $O
