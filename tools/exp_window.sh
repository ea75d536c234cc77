# window-ring view FFT (tuning gen_window) at config 4 (signals in HBM): parity test, bench
# lines per look-ahead, and the FFT kernel's ncu time / DRAM bytes
O=gpurun_out/win; mkdir -p $O
python -m pytest tests/test_gpu_parity.py -q -x -k "window_ring" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -n 3 $O/pytest.log
for w in 0 8 16 24 32 0 16; do
  SFDT_GEN_WINDOW=$w timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4_w$w.json 2>>$O/err
done
for f in $O/cfg4_w*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4))"; done
for w in 0 16; do
  SFDT_GEN_WINDOW=$w timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft -c 4 --csv --log-file $O/ncu_w$w.csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 1 > /dev/null 2>>$O/err
  grep -E "k_fft" $O/ncu_w$w.csv | awk -F'","' '{print $5, $(NF-2), $(NF)}' | tail -n 6
done
