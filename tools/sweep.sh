#!/bin/bash
# Round measurement sweep (GPU box, one GPU): every BASELINE.json workload
# through bench.py, one JSON line each, into gpurun_out/sweep/.
mkdir -p gpurun_out/sweep
O=gpurun_out/sweep
python bench.py --config cfg1 --steps 50 --warmup 5 > $O/bench_cfg1.json 2> $O/cfg1.err
python bench.py --config cfg2 > $O/bench_cfg2.json 2> $O/cfg2.err
python bench.py --config cfg3 --steps 10 --warmup 3 > $O/bench_cfg3.json 2> $O/cfg3.err
python bench.py --config cfg4 --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/cfg4.err
python bench.py --config cfg2 --solver iterative --no-cpu --steps 20 --warmup 3 > $O/it.json 2> $O/it.err
python bench.py --config cfg2 --dtype c64 --no-cpu --steps 20 --warmup 3 > $O/c64.json 2> $O/c64.err
python bench.py --config cfg3 --mu 4 --no-cpu --no-e2e --steps 10 --warmup 3 > $O/cfg3_mu4.json 2> $O/cfg3_mu4.err
for k in 64 256 1024 4096 16384; do
  python bench.py --config cfg5 --k $k --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c5e_$k.json 2> $O/c5e_$k.err
  python bench.py --config cfg5 --cfg5-general --k $k --no-cpu --no-e2e --steps 5 --warmup 3 > $O/c5g_$k.json 2> $O/c5g_$k.err
done
python bench.py --config cfg4 --no-prune --no-cpu --no-e2e --steps 5 --warmup 3 > $O/cfg4_noprune.json 2> $O/cfg4_noprune.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_cfg2.json 2> $O/ref_cfg2.err
python bench.py --impl reference --config cfg4 --steps 2 --warmup 1 > $O/ref_cfg4.json 2> $O/ref_cfg4.err
for k in 64 256 1024; do
  python bench.py --config cfg5 --cfg5-general --no-prune --k $k --no-cpu --no-e2e --steps 5 --warmup 3 > $O/c5g_noprune_$k.json 2> $O/c5g_noprune_$k.err
done
python bench.py --config cfg5 --k 1024 --dtype c64 --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c5e_1024_c64.json 2> $O/c5e_1024_c64.err
for f in $O/*.json; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1])
    print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],3), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))
except Exception as e: print('$f', 'ERR', e)
"; done
