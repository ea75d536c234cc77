O=gpurun_out/exp2; mkdir -p $O
python -m pytest tests -m gpu -q -x -k "heavy_bins or solve_graph or general" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for ov in 1 0 1 0; do
  SFDT_GEN_OVERLAP=$ov python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4_ov$ov.json 2>>$O/err
  SFDT_GEN_OVERLAP=$ov python bench.py --config cfg5 --cfg5-general --k 16384 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g_ov$ov.json 2>>$O/err
  SFDT_GEN_OVERLAP=$ov python bench.py --config cfg5 --cfg5-general --k 1024 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g1k_ov$ov.json 2>>$O/err
done
tail -3 $O/pytest.log
for f in $O/*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4))"; done
