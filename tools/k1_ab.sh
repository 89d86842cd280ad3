for lib in variants/lib_*.so; do echo "== $lib"; PFT_LIB=$lib QT=k1ab python tools/quick_time.py 2>&1 | grep -v Warn | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['label'], d['us'], d['k1_us'])
"; for pp in 256 512; do PFT_LIB=$lib timeout 300 python bench.py --config c3 --steps 10 --no-cpu --no-e2e --p $pp 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('C3', $pp, round(d['value']), round(d['ms_per_step'],3))"; done; done
