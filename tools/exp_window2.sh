O=gpurun_out/win2; mkdir -p $O
for w in 16 1016 2016; do
  SFDT_GEN_WINDOW=$w timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft -c 2 --csv --log-file $O/ncu_w$w.csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 1 > /dev/null 2>>$O/err
  echo "== $w"; grep -E "k_fft" $O/ncu_w$w.csv | awk -F'","' '{print $(NF-2), $(NF)}' | tail -n 3
done
