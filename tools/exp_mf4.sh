O=gpurun_out/exp9; mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x -k "general or matched or heavy or prune" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for k in 64 256 1024 4096; do
  python bench.py --config cfg5 --cfg5-general --k $k --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g_$k.json 2>>$O/err
done
python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4.json 2>>$O/err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gen_mf" -c 2 --csv python bench.py --config cfg5 --cfg5-general --k 64 --no-cpu --no-e2e --steps 1 --warmup 0 > $O/ncu_mf.csv 2>/dev/null
tail -3 $O/pytest.log
for f in $O/*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4), d['parity_sample']['supports_equal'], d['parity_sample']['max_rel'])"; done
grep -h gpu__time $O/ncu_mf.csv | awk -F, '{print $NF}'
