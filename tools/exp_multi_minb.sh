# k_decode_multi resident CTAs per SM (variants/lib_mminbN.so: SFDT_MULTI_MINB; default 6) at config 2 / config 3
O=gpurun_out/mminb; mkdir -p $O
for v in base mminb2 mminb3 mminb4 mminb8; do
  L=""; [ $v != base ] && L=$PWD/variants/lib_$v.so
  for c in "--config cfg2" "--config cfg3"; do
    n=$(echo $c | tr -d ' -')
    SFDT_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_decode_multi" -c 4 --csv --log-file $O/ncu_${v}_$n.csv python bench.py $c --no-cpu --no-e2e --steps 1 --warmup 1 > /dev/null 2>>$O/err
    echo "== $v $c"; grep -E "k_decode" $O/ncu_${v}_$n.csv | awk -F'","' '{print substr($5,1,24), $(NF)}' | tail -n 4 | tr '\n' ' '; echo
  done
done
