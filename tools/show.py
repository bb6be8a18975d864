import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().split('\n')[-1])
        sm = {k: round(v, 2) for k, v in d['stage_ms'].items() if v}
        print(f.split('/')[-1], 'ms/step', round(d['ms_per_step'], 2), 'value %.3g' % d['value'], 'frac %.3f' % d['roofline']['frac'],
              'rebuilds', d.get('rebuilds_in_timed_region'), 'rebuild_ms', round(d.get('rebuild_ms', 0), 2), sm)
    except Exception as e:
        print(f, 'ERR', open(f).read()[-800:])
