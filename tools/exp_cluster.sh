O=gpurun_out/exp6; mkdir -p $O
for c in 0 8 4 2 0 8; do
  SFDT_FFT_CLUSTER=$c python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4_c$c.json 2>>$O/err_$c
done
for c in 0 8; do
  SFDT_FFT_CLUSTER=$c python bench.py --config cfg2 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg2_c$c.json 2>>$O/err_$c
  SFDT_FFT_CLUSTER=$c python bench.py --config cfg5 --cfg5-general --k 1024 --no-cpu --no-e2e --steps 5 --warmup 3 >> $O/c5g1k_c$c.json 2>>$O/err_$c
  SFDT_FFT_CLUSTER=$c timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_fft_views -c 2 --csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 0 > $O/ncu_c$c.csv 2>/dev/null
done
for f in $O/*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4), d.get('parity_sample'), (d['roofline'].get('random_access') or {}).get('achieved_g_per_s'))"; done
for c in 0 8; do echo c$c; grep -h -E "gpu__time|dram__bytes" $O/ncu_c$c.csv | awk -F, '{print $(NF-2), $NF}'; done
tail -3 $O/err_8
