for m in 0 1 3; do
 SFDT_A16_LD=$m ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:k_fft_large_a16 -c 2 --csv --log-file /tmp/m$m.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 0 --config cfg5 --cfg5-general --k 16384 > /dev/null 2>&1
 echo "LD=$m"; grep -E "gpu__time|dram__bytes|hit_rate" /tmp/m$m.csv | awk -F'","' '{print $(NF-2), $NF}' | head -6
done
