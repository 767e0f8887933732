# pipelined host entry: e2e vs compute lanes (IDK_HOST_LANES), same box
for r in 1 2; do for L in 1 2 8; do for c in cfg1 cfg2; do IDK_HOST_LANES=$L python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes $L $c e2e', round(d['e2e']['value'],1))"; done; done; done
