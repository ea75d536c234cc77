# pass A of every large view through k_fft_large_a16 (L = 2^13..2^16 too): parity test, A/B bench lines
# (SFDT_FFT_SPLIT=1 = k_fft_large_a + register passes, the previous plan for these L) and launch lists
O=gpurun_out/a16all; mkdir -p $O
python -m pytest tests/test_gpu_parity.py -q -x -k "large_view or fft_large or cfg5 or io_cli" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log; tail -n 3 $O/pytest.log
python -m pytest tests/test_io_cli.py tests/test_gpu_configs.py -q -x -m gpu >> $O/pytest2.log 2>&1; echo rc=$? >> $O/pytest2.log; tail -n 3 $O/pytest2.log
run() { # name, args
  for sp in 1 0 1 0; do
    SFDT_FFT_SPLIT=$sp python bench.py $2 --no-cpu --no-e2e --steps 10 --warmup 3 2>>$O/err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 split=$sp', round(d['value'],1), round(d['ms_per_step'],4))"
  done
}
run c5e_16384 "--config cfg5 --k 16384"
run c5e_4096 "--config cfg5 --k 4096"
run cfg3_mu4 "--config cfg3 --mu 4"
run c5g_1024 "--config cfg5 --cfg5-general --k 1024"
for c in "--config cfg5 --k 16384" "--config cfg3" "--config cfg3 --mu 4"; do
  n=$(echo $c | tr -d ' -'); 
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file $O/launches_$n.csv python bench.py $c --no-cpu --no-e2e --steps 1 --warmup 1 > /dev/null 2>>$O/err
  echo "== $c"; python tools/launches.py $O/launches_$n.csv 2
done
