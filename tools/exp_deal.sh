O=gpurun_out/exp3; mkdir -p $O
python -m pytest tests/test_gpu_parity.py -q -x -k "heavy_bins or noprune or general_grid or cfg5" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for dl in 8 0 2 4 32 8 0; do
  SFDT_GEN_DEAL=$dl python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4_d$dl.json 2>>$O/err
done
for dl in 8 0; do
  SFDT_GEN_DEAL=$dl python bench.py --config cfg5 --cfg5-general --k 16384 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g_d$dl.json 2>>$O/err
  SFDT_GEN_DEAL=$dl python bench.py --config cfg5 --cfg5-general --k 4096 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g4k_d$dl.json 2>>$O/err
  SFDT_GEN_DEAL=$dl python bench.py --config cfg4 --no-prune --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/cfg4np_d$dl.json 2>>$O/err
  SFDT_GEN_DEAL=$dl ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gen_bins -c 3 --csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 1 > $O/ncu_bins_d$dl.csv 2>/dev/null
done
tail -3 $O/pytest.log
for f in $O/*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4))"; done
grep -h gpu__time $O/ncu_bins_d*.csv | awk -F, '{print $NF}'
