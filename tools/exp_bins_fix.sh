O=gpurun_out/binsfix; mkdir -p $O
python -m pytest tests -m gpu -q -x -k "general or dropin or reference_suite or scale" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log; tail -n 4 $O/pytest.log
SFDT_GEN_OVERLAP=0 SFDT_LIB=$PWD/variants/lib_prof.so timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 0 > $O/prof.txt 2>$O/err
grep BIN $O/prof.txt | sed 's/.*cyc=\([0-9]*\) .*/\1 &/' | sort -n | tail -n 6
for i in 1 2; do timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 --warmup 3 >> $O/cfg4.json 2>>$O/err; done
python -c "
import json
for l in open('$O/cfg4.json'):
    d=json.loads(l); print(round(d['value'],1), round(d['ms_per_step'],4))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gen_bins|k_gen_sp1" -c 4 --csv --log-file $O/ncu.csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 1 > /dev/null 2>>$O/err
grep -E "k_gen" $O/ncu.csv | awk -F'","' '{print substr($5,1,24), $(NF)}' | tail -n 4
