O=gpurun_out/exp7; mkdir -p $O
python -m pytest tests/test_gpu_parity.py -q -x -k "prune_four_lanes or general_grid or cfg5 or heavy_bins" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for l in 4 1 4 1; do
  SFDT_GEN_PRUNE_LANES=$l python bench.py --config cfg5 --cfg5-general --k 64 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g64_l$l.json 2>>$O/err
done
python bench.py --config cfg5 --cfg5-general --k 256 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g256.json 2>>$O/err
python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4.json 2>>$O/err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gen_prune -c 2 --csv python bench.py --config cfg5 --cfg5-general --k 64 --no-cpu --no-e2e --steps 1 --warmup 0 > $O/ncu_prune4.csv 2>/dev/null
tail -3 $O/pytest.log
for f in $O/*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4), d['parity_sample'])"; done
grep -h gpu__time $O/ncu_prune4.csv | awk -F, '{print $NF}'
