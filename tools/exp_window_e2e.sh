# window-ring gather (tuning gen_window) on the zero-copy host path: the six consecutive shifts of a
# d-block become ONE 96-B PCIe read instead of six 16-B reads from six different CTAs.
# gen_window: 0 off, -1 auto (16 for host-mapped x, no fetch-size hint), -2 auto with the L2::64B hint
O=gpurun_out/wine2e; mkdir -p $O
python -m pytest tests -m gpu -q -x -k "zero_copy or host_batch or window or general" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log; tail -n 3 $O/pytest.log
for w in 0 -1 -2 -1 -2; do
  SFDT_GEN_WINDOW=$w python bench.py --config cfg4 --no-cpu --steps 3 --warmup 1 2>>$O/err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 window=$w value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['pcie']['frac'],3))"
done
for ch in 128 512 1024; do
  python bench.py --config cfg4 --no-cpu --steps 3 --warmup 1 --e2e-chunk $ch 2>>$O/err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 auto chunk=$ch value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['pcie']['frac'],3))"
done
