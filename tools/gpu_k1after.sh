# overlap variants: where K1 of step k+1 starts, and the free-SM count
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
for a in staged start; do for f in 0 8 16; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --k1-after $a --free-sms $f > gpurun_out/ka_${a}_$f.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ka_${a}_$f.json'));print('$a', $f, round(d['value']/1e6,1), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})"
done; done
