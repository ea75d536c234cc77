O=gpurun_out/gate; mkdir -p $O
python -m pytest tests -m gpu -q -x -k "cooperative or latency_path or cfg3 or cfg2 or golden or duplicate or noniter or exact" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log; tail -n 3 $O/pytest.log
for c in "--config cfg3" "--config cfg2" "--config cfg5 --k 16384" "--config cfg3 --mu 4" "--config cfg5 --k 4096"; do
  for i in 1 2; do
  python bench.py $c --no-cpu --no-e2e --steps 10 --warmup 3 2>>$O/err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['value'],1), round(d['ms_per_step'],4), d.get('gpu_launches'))"
  done
done
