python bench.py > gpurun_out/s24_bench.json 2> gpurun_out/s24_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/s24_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms/step', d['ms_per_step'], 'roofline', d['roofline']['frac'], d['roofline']['achieved'], 'setup', d.get('setup_roofline',{}).get('frac'), 'e2e', d['e2e']['value'])
ns=d['north_star']; print({k:(v.get('ms'), v.get('frac_of_peak')) for k,v in ns.items() if isinstance(v,dict)})
"
timeout 900 python tools/report.py > gpurun_out/s24_report.md 2>&1; tail -20 gpurun_out/s24_report.md
