# Grouped-sketch batch experiments (cfg2): chunk size, lane priority, grouped on/off.
python -m pytest tests/test_gpu_id.py -x -q -k "batch" > gpurun_out/t_batch.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t_batch.log
run() { echo "== $*"; env "$@" python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['ms_per_step'], {k: round(v,4) for k,v in d['stages_ms_per_step'].items()})"; }
run IDK_BATCH_GROUPED=0
run IDK_BATCH_GROUPED=0 IDK_LANE_PRIO=0
run IDK_BATCH_CHUNK=2
run IDK_BATCH_CHUNK=4
run IDK_BATCH_CHUNK=8
run IDK_BATCH_CHUNK=16
run IDK_BATCH_CHUNK=4 IDK_LANE_PRIO=0
run IDK_BATCH_CHUNK=4 IDK_GEMM_SPLITS=1
run IDK_BATCH_CHUNK=4 IDK_GEMM_SPLITS=2
run IDK_BATCH_CHUNK=8 IDK_GEMM_SPLITS=1
