O=gpurun_out/exp1; mkdir -p $O
for h in 0 1 2 3; do
  SFDT_GATHER_HINT=$h python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 > $O/cfg4_h$h.json 2>$O/cfg4_h$h.err
  SFDT_GATHER_HINT=$h python bench.py --config cfg5 --cfg5-general --k 16384 --no-cpu --no-e2e --steps 5 --warmup 3 > $O/c5g_h$h.json 2>$O/c5g_h$h.err
  SFDT_GATHER_HINT=$h python bench.py --config cfg2 --no-cpu --no-e2e --steps 10 --warmup 3 > $O/cfg2_h$h.json 2>$O/cfg2_h$h.err
done
for h in 0 1 2 3; do
  SFDT_GATHER_HINT=$h timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft -c 3 --csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 0 > $O/ncu_h$h.csv 2>/dev/null
done
for f in $O/*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4))"; done
