# A/B/C... of library builds on one box (IDK_LIB_PATH), alternating, bench stage times.
#   bash tools/ab_variants.sh "cfg4 cfg5" paper_2105_07076_b200/ab/F0.so paper_2105_07076_b200/ab/F1.so ...
# The last build also runs the core GPU tests first.
cfgs=$1; shift
last=${@: -1}
IDK_LIB_PATH=$last timeout 900 python -m pytest tests -x -q -m gpu -k "qr or id or rid or config or edge" -p no:cacheprovider 2>&1 | tail -1
for r in 1 2 3; do for v in "$@"; do for c in $cfgs; do
  IDK_LIB_PATH=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $v)', '$c', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stages_ms_per_step'].items()})"
done; done; done
