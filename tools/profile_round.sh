#!/usr/bin/env bash
# Round profile capture (run on the GPU box from the repo root via gpurun):
# bench line, reference arm, ncu launch list of the same bench command, and a
# full ncu capture of the main kernels of one c2 compress.  Outputs land in
# gpurun_out/; tools/summarize_round.py turns them into profiles/.
set -u
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench_err.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref_err.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"syrk_kernel|syrk_reduce|ttm_kernel|tk_cluster|ac_kernel|householder_dataflow|crossing_kernel|emit_kernel|stats_kernel" \
    -c 24 -o gpurun_out/full python tools/compress_once.py --warmup 0 > gpurun_out/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv \
    python tools/decompress_once.py --steps 1 --warmup 0 > gpurun_out/dec_ncu.log 2>&1
echo done
