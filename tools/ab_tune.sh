for t in 0 1; do
MSSZ_TUNE=$t MSSZ_TRACE=1 timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > gpurun_out/ab_$t.json 2> gpurun_out/ab_$t.err
python - $t <<'PY'
import re,sys,json
t=sys.argv[1]
small=big=0; ph=[0,0,0]
lines=open(f"gpurun_out/ab_{t}.err").read().splitlines()
# second half of trace = timed step (warmup 1 + step 1)
half=[i for i,l in enumerate(lines) if 'C kind=0' in l]
start=half[len(half)//2] if half else 0
for l in lines[start:]:
    m=re.search(r'small_ms=([\d.]+) big_ms=([\d.]+)',l)
    if m: small+=float(m.group(1)); big+=float(m.group(2))
    m=re.search(r'big phases fix=([\d.]+) frontier=([\d.]+) rebuild=([\d.]+)',l)
    if m:
        for i in range(3): ph[i]+=float(m.group(i+1))
d=json.loads(open(f"gpurun_out/ab_{t}.json").read().strip().splitlines()[-1])
print("tune",t,"ms/step %.1f"%d["ms_per_step"],"small %.1f big %.1f phases %s"%(small,big,[round(x,1) for x in ph]))
PY
done
