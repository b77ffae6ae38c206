for i in 1 2; do timeout -s KILL 300 python bench.py 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks'])"; done
