O=gpurun_out/exp4; mkdir -p $O
python -m pytest tests/test_gpu_parity.py -q -x -k "heavy_bins or noprune or general_grid" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for sp in 3 0 2 3 0; do
  SFDT_GEN_SPLIT=$sp python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4_s$sp.json 2>>$O/err
done
for sp in 3 0; do
  SFDT_GEN_SPLIT=$sp ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gen_bins -c 3 --csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 1 > $O/ncu_bins_s$sp.csv 2>/dev/null
  SFDT_GEN_SPLIT=$sp python bench.py --config cfg4 --no-prune --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/cfg4np_s$sp.json 2>>$O/err
done
tail -3 $O/pytest.log
for f in $O/*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4))"; done
for sp in 3 0; do echo s$sp; grep -h gpu__time $O/ncu_bins_s$sp.csv | awk -F, '{print $NF}'; done
