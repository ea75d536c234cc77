# host-mapped signals: window gather kernel + FFT from its buffer (any L) vs the ring (L = 4096) vs per-view gather
O=gpurun_out/wing; mkdir -p $O
python -m pytest tests/test_gpu_api.py -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log; tail -n 3 $O/pytest.log
e2e() { python bench.py $2 --no-cpu --steps 3 --warmup 1 2>>$O/err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d.get('e2e') or {}; print('$1', 'value', round(d['value'],1), 'e2e', e.get('value'), (e.get('pcie') or {}).get('frac'))"; }
for w in -1 -4 0 -1 -4; do SFDT_GEN_WINDOW=$w e2e "cfg4 window=$w" "--config cfg4"; done
for k in 64 256 1024; do
  for w in 0 -1; do SFDT_GEN_WINDOW=$w e2e "c5g k=$k window=$w" "--config cfg5 --cfg5-general --k $k"; done
done
