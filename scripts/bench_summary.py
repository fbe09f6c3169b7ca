import json,sys
for l in sys.stdin:
    if not l.startswith('{'): continue
    j=json.loads(l)
    print(j['config']['workload'][:3], 'steps/s %.1f ms/step %.3f refresh %s e2e %s launches %s' % (j['value'], j['ms_per_step'], j.get('refresh_ms'), (j.get('e2e') or {}).get('value'), j.get('gpu_launches')))
    print('  phases', {k:(v['ms_total'],v['count']) for k,v in (j.get('phases') or {}).items()})
    print('  kernels', {k:(v['ms_total'],v['launches'],v['avg_us']) for k,v in (j.get('kernels') or {}).items()})
