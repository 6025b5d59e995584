for v in 0 1; do
TCB_NO_EARLY_PREP=$v TCB_TIMELINE=1 timeout 300 python tools/compress_once.py --warmup 3 --steps 1 > gpurun_out/ctl$v.log 2>&1
done
for v in 0 1; do TCB_NO_EARLY_PREP=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ep$v.json 2>/dev/null; done
