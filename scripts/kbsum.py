"""Summarise a kbench log with '== label' separators: label | case ms | ..."""
import json
import sys
for l in open(sys.argv[1]):
    if l.startswith('=='):
        print('\n' + l.strip(), end=' | ')
    elif l.startswith('{'):
        d = json.loads(l)
        print(d['case'], d['ms'], end=' | ')
    elif l.strip():
        print(l.strip()[:120])
print()
