# A/B of the large-view FFT plans (SFDT_FFT_SPLIT=1: stage-split 4+3
# register passes; 0: register-blocked pass A + one pass B), launch lists at
# config 5 general K=2^14 (L=2^19) and exact K=2^14 (L=2^16) / mu=1 cfg3-like
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "large or fft" 2>&1 | tail -2 > gpurun_out/r2_exp.log
timeout 900 python -m pytest tests/test_gpu_dropin.py -q -x -k "aliased" 2>&1 | tail -2 >> gpurun_out/r2_exp.log
for v in 1 0; do
 for c in "--config cfg5 --cfg5-general --k 16384" "--config cfg5 --cfg5-general --k 4096" "--config cfg3 --mu 4"; do
  SFDT_FFT_SPLIT=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_fft --csv --log-file /tmp/l.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 $c > /dev/null 2>&1
  echo "PIPE=$v $c" >> gpurun_out/r2_exp.log; python tools/launches.py /tmp/l.csv 2 >> gpurun_out/r2_exp.log
 done
 SFDT_FFT_SPLIT=$v python bench.py --no-cpu --no-e2e --steps 5 --warmup 2 --config cfg5 --cfg5-general --k 16384 > gpurun_out/r2_c5g16k_split$v.json 2>/dev/null
done
