mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --config $CFG --steps $ST --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', '$*', round(d['value'],1), round(d['kernel_ms']['taylor'],4))"; }
for rep in 1 2; do
CFG=C3 ST=100 run GS_X=0
CFG=C3 ST=100 run GS_GRID=144
CFG=C3 ST=100 run GS_GRID=128
CFG=C3 ST=100 run GS_LOCK=0
CFG=C3 ST=100 run GS_LOCK_C0=6
CFG=C3 ST=100 run GS_LOCK_C0=1.5
CFG=C4 ST=10 run GS_X=0
CFG=C4 ST=10 run GS_GRID=144
CFG=C4 ST=10 run GS_LOCK_C0=6
done
