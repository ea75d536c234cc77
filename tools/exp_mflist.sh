O=gpurun_out/exp8; mkdir -p $O
python -m pytest tests/test_gpu_parity.py -q -x -k "prune_four_lanes or general_grid or cfg5 or heavy_bins or matched" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for m in auto 4096 auto 4096; do
  if [ $m = auto ]; then E=""; else E="SFDT_GEN_MF_LIST=$m"; fi
  env $E python bench.py --config cfg5 --cfg5-general --k 64 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g64_$m.json 2>>$O/err
done
python bench.py --config cfg5 --cfg5-general --k 256 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g256.json 2>>$O/err
python bench.py --config cfg5 --cfg5-general --k 1024 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g1024.json 2>>$O/err
python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4.json 2>>$O/err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gen_(mf|prune|bins)" -c 6 --csv python bench.py --config cfg5 --cfg5-general --k 64 --no-cpu --no-e2e --steps 1 --warmup 0 > $O/ncu_c5g64.csv 2>/dev/null
tail -3 $O/pytest.log
for f in $O/*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4), d['parity_sample']['supports_equal'])"; done
grep -h gpu__time $O/ncu_c5g64.csv | awk -F'","' '{print $5, $NF}' | cut -c1-60
