#!/bin/bash
# Launch lists (ncu gpu__time_duration per kernel, cold-cache, serialised) of
# the main workloads; run on the GPU box through gpurun.  $1 = tag.
T=${1:-r02}
mkdir -p gpurun_out
B="python bench.py --no-cpu --no-e2e --steps 1 --warmup 1"
NM="ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv"
$NM --log-file gpurun_out/${T}_launches_cfg2.csv $B > /dev/null 2>&1
$NM --log-file gpurun_out/${T}_launches_cfg4.csv $B --config cfg4 > /dev/null 2>&1
$NM --log-file gpurun_out/${T}_launches_c5g16k.csv $B --config cfg5 --cfg5-general --k 16384 > /dev/null 2>&1
$NM --log-file gpurun_out/${T}_launches_c5e16k.csv $B --config cfg5 --k 16384 > /dev/null 2>&1
for f in gpurun_out/${T}_launches_*.csv; do echo "== $f"; python tools/launches.py $f 2; done
