#!/bin/bash
# Config 4 view FFT: radix-16 register-blocked kernel vs k_fft_views (SFDT_FFT_SPLIT=2) and
# the L2 prefetch-ahead of the gather (sfdt_tuning.gen_prefetch = signals ahead).
O=gpurun_out/pf; mkdir -p $O
run() {  # tag, env...
  tag=$1; shift
  env "$@" python bench.py --config cfg4 --no-cpu --no-e2e --steps 20 --warmup 3 > $O/cfg4_$tag.json 2>/dev/null
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft -c 2 --csv --log-file $O/ncu_$tag.csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 1 > /dev/null 2>&1
  echo "$tag $(python -c "import json; d=json.load(open('$O/cfg4_$tag.json')); print(round(d['value']), round(d['ms_per_step'],4), d.get('parity_sample'))") $(grep -E 'gpu__time_duration|dram__bytes' $O/ncu_$tag.csv | tail -3 | awk -F'","' '{print $(NF-2), $(NF)}' | tr -d '"' | tr '\n' ' ')"
}
run r8 SFDT_FFT_SPLIT=2
run r16 SFDT_FFT_SPLIT=0
for m in ${MODES:-8 16 20 24 32 48}; do run r16_pf$m SFDT_GEN_PREFETCH=$m; done
