timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "large or fft or cfg5_general or long_view or closed_form" 2>&1 | tail -2 > gpurun_out/r2_e4.log
for c in "--config cfg5 --cfg5-general --k 16384" "--config cfg5 --cfg5-general --k 4096" "--config cfg4"; do
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file /tmp/l.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 $c > /dev/null 2>&1
  echo "$c" >> gpurun_out/r2_e4.log; python tools/launches.py /tmp/l.csv 2 >> gpurun_out/r2_e4.log
  python bench.py --no-cpu --no-e2e --steps 5 --warmup 2 $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', round(d['value']), d['ms_per_step'], d['parity_sample'])" >> gpurun_out/r2_e4.log
done
