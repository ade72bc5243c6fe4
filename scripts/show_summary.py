import json, sys
for d in json.load(open(sys.argv[1])):
    print(d['kernel'])
    for k, v in d.items():
        if k not in ('kernel', 'stalls_per_issue'):
            print('   ', k, v)
    print('   stalls', {k: round(v, 2) for k, v in d['stalls_per_issue'].items()})
