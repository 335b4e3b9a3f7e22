python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
for a in staged start; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --k1-after $a > gpurun_out/e2e_$a.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/e2e_$a.json'));print('$a', round(d['value']/1e6,1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3))"
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload bursty > gpurun_out/bursty.json 2>gpurun_out/bursty.err; echo bursty rc=$?
python -c "import json;d=json.load(open('gpurun_out/bursty.json'));print('bursty', round(d['value']/1e6,1), round(d['ms_per_step'],3), d['phase_ms'], 'e2e', d['e2e'] and round(d['e2e']['value']/1e6,1))"
