# resident CTAs per SM of k_decode_a1_dense (SFDT_A1D_MINB) and k_iter_decode (SFDT_ITER_MINB): ncu kernel times at config 2
O=gpurun_out/docc; mkdir -p $O
for v in base a1d3 a1d8; do
  L=""; [ $v != base ] && L=$PWD/variants/lib_$v.so
  SFDT_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_decode_a1_dense" -c 3 --csv --log-file $O/ncu_$v.csv python bench.py --no-cpu --no-e2e --steps 2 --warmup 1 > /dev/null 2>>$O/err
  echo "== $v a1_dense: $(grep -E 'k_decode' $O/ncu_$v.csv | awk -F'\",\"' '{print $(NF)}' | tr -d '\"' | tr '\n' ' ')"
done
for v in base it2 it3; do
  L=""; [ $v != base ] && L=$PWD/variants/lib_$v.so
  SFDT_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_iter_decode" -c 8 --csv --log-file $O/ncui_$v.csv python bench.py --solver iterative --no-cpu --no-e2e --steps 1 --warmup 1 > /dev/null 2>>$O/err
  echo "== $v iter_decode<0..3> x2: $(grep -E 'k_iter_decode' $O/ncui_$v.csv | awk -F'\",\"' '{print $(NF)}' | tr -d '\"' | tr '\n' ' ')"
done
