# k_gen_bins resident CTAs per SM (variants/lib_minb{3,4}.so: SFDT_BINS_MINB) at config 4
O=gpurun_out/minb; mkdir -p $O
for v in base minb3 minb4 base minb4; do
  L=""; [ $v != base ] && L=$PWD/variants/lib_$v.so
  SFDT_LIB=$L timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4_$v.json 2>>$O/err
done
for f in $O/cfg4_*.json; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],4))"; done
for v in base minb3 minb4; do
  L=""; [ $v != base ] && L=$PWD/variants/lib_$v.so
  SFDT_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gen_bins|k_gen_sp1" -c 4 --csv --log-file $O/ncu_$v.csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 1 > /dev/null 2>>$O/err
  echo "== $v"; grep -E "k_gen" $O/ncu_$v.csv | awk -F'","' '{print substr($5,1,24), $(NF)}' | tail -n 4
done
