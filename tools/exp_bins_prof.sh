O=gpurun_out/binsprof; mkdir -p $O
SFDT_GEN_OVERLAP=0 SFDT_LIB=$PWD/variants/lib_prof.so timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --steps 1 --warmup 0 > $O/out.txt 2>$O/err
grep -c BIN $O/out.txt
grep BIN $O/out.txt | sort -t= -k9 -n | awk '{print}' | sort -k9 | tail -n 5
python - <<'PY'
import re,collections
rows=[]
for l in open('gpurun_out/binsprof/out.txt'):
    if l.startswith('BIN'):
        d=dict(kv.split('=') for kv in l.split()[1:])
        rows.append({k:int(v) for k,v in d.items()})
rows.sort(key=lambda r:-r['cyc'])
print(len(rows))
for r in rows[:25]: print(r)
import statistics
samp=[r for r in rows if r['q']%64==0]
print('sample n',len(samp),'median cyc',statistics.median(r['cyc'] for r in samp))
c=collections.Counter((r['a'],r['minnorm']>0) for r in rows if r['cyc']>150000)
print(c)
PY
