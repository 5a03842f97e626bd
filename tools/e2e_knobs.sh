for S in 8 12 16 24; do echo "S=$S"; FAGP_GRAM_SUBRANGES=$S python bench.py --no-cpu-baseline 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('  device', d['ms_per_step'], 'e2e', round(d['e2e']['ms_per_step'],3))
    elif 'e2e step' in l: print('  ', l.strip())
"; done
for C in 3 4 8; do echo "PC=$C"; FAGP_PREDICT_CHUNKS=$C python bench.py --no-cpu-baseline 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('  device', d['ms_per_step'], 'e2e', round(d['e2e']['ms_per_step'],3))
"; done
