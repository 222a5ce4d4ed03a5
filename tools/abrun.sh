mkdir -p gpurun_out
for rep in 1 2; do for v in V2 V3 V4; do
cp tools/lib$v.so paper_2402_02273_b200/libgliosim_b200.so
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), round(d['roofline']['avg_launch_ms'],3))"
done; done
