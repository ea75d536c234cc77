O=gpurun_out/exp5; mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x -k "heavy_bins or noprune or general or graph" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for v in 1 0 1 0; do
  SFDT_GEN_PRUNE2=$v python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4_p$v.json 2>>$O/err
  SFDT_GEN_PRUNE2=$v python bench.py --config cfg4 --no-prune --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/cfg4np_p$v.json 2>>$O/err
  SFDT_GEN_PRUNE2=$v python bench.py --config cfg5 --cfg5-general --k 4096 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g4k_p$v.json 2>>$O/err
done
SFDT_GEN_PRUNE2=1 python bench.py --config cfg5 --cfg5-general --k 16384 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g16k_p1.json 2>>$O/err
SFDT_GEN_PRUNE2=1 python bench.py --config cfg5 --cfg5-general --k 64 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g64_p1.json 2>>$O/err
tail -3 $O/pytest.log
for f in $O/*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4))"; done
