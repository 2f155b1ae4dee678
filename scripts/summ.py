import json, sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d = json.loads(line)
        print("VALUE", d['value'], "e2e", d.get('e2e', {}).get('value'), [(k['label'], k['ms']) for k in d['kernels']])
