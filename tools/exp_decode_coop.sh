#!/bin/bash
# Cooperative multi-collision decode A/B (sfdt_tuning.decode_coop): bench lines and
# ncu launch lists per mode.  Run on the GPU box through gpurun.
O=gpurun_out/coop; mkdir -p $O
python -m pytest tests/test_gpu_parity.py -q -x -k "cooperative_decode" 2>&1 | tail -5 > $O/pytest.log
for m in 0 1 2 3; do
  SFDT_DECODE_COOP=$m python bench.py --config cfg1 --no-cpu --no-e2e --steps 50 --warmup 5 > $O/cfg1_m$m.json 2>/dev/null
  SFDT_DECODE_COOP=$m python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 > $O/cfg2_m$m.json 2>/dev/null
done
for m in 0 1; do
  SFDT_DECODE_COOP=$m ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file $O/l_cfg1_m$m.csv python bench.py --config cfg1 --no-cpu --no-e2e --graph off --steps 2 --warmup 2 > /dev/null 2>&1
done
for m in 0 2; do
  SFDT_DECODE_COOP=$m ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_dec --csv --log-file $O/l_cfg2_m$m.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 > /dev/null 2>&1
done
cat $O/pytest.log
for f in $O/cfg*.json; do echo $f $(python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d['ms_per_step'])"); done
for f in $O/l_*.csv; do echo == $f; python tools/launch_times.py $f | grep dec | tail -4; done
