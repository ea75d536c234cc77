for pre in 0 1; do
 SFDT_B16_PRE=$pre ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fft_large -c 4 --csv --log-file /tmp/b$pre.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 0 --config cfg5 --cfg5-general --k 16384 > /dev/null 2>&1
 echo "B16_PRE=$pre"; python tools/launches.py /tmp/b$pre.csv 2
done
SFDT_B16_PRE=0 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fft_large -c 4 --csv --log-file /tmp/b4k.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 0 --config cfg5 --cfg5-general --k 4096 > /dev/null 2>&1
echo "K=4096 PRE=0"; python tools/launches.py /tmp/b4k.csv 2
