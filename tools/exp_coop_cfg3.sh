O=gpurun_out/coop3; mkdir -p $O
for m in 2 0 1 3 2 0; do
  SFDT_DECODE_COOP=$m python bench.py --config cfg3 --no-cpu --no-e2e --steps 10 --warmup 3 2>>$O/err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3 coop=$m', round(d['value'],1), round(d['ms_per_step'],4))"
done
for m in 2 0 1 3; do
  SFDT_DECODE_COOP=$m python bench.py --config cfg5 --k 16384 --no-cpu --no-e2e --steps 10 --warmup 3 2>>$O/err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5e16k coop=$m', round(d['value'],1), round(d['ms_per_step'],4))"
done
