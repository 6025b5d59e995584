#!/usr/bin/env bash
# Round profile capture (run on the GPU box from the repo root via gpurun):
# bench line, reference arm, ncu launch list of the bench command and of one
# c5 compress, and a full ncu capture of the main kernels of one c5 compress.
# Outputs land in gpurun_out/; tools/summarize_round.py turns them into profiles/.
set -u
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench_err.log
[ -n "${SKIP_REF:-}" ] || python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref_err.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launches.log 2>&1
C5_PROFILE=1 C5_NO_DEC=1 C5_ITERS=2 ncu --profile-from-start off --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/launches.csv python tools/c5_once.py 1e-2 \
    > gpurun_out/ncu_c5.log 2>&1
C5_PROFILE=1 C5_NO_DEC=1 C5_ITERS=2 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"oz_mma_kernel|oz_split_rows_blk|oz_split_cols_blk|ex_plane_kernel|ex_walk_kernel|ac_range_kernel|ac_code_kernel|sc_emit|tridiag_coop|dm_decode" \
    -c 16 -o gpurun_out/full python tools/c5_once.py 1e-2 > gpurun_out/ncu_full.log 2>&1
C5_PROFILE=1 C5_NO_DEC=1 C5_ITERS=2 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"ex_plane_kernel|sc_emit_kernel|ac_range_kernel|ac_code_kernel|ex_walk_kernel|dm_decode" \
    -c 10 -o gpurun_out/full_enc python tools/c5_once.py 1e-2 > gpurun_out/ncu_full_enc.log 2>&1
# gpurun brings back at most 64 MiB: keep the raw metric pages, not the reports
for r in full full_enc; do
    ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2> /dev/null
    rm -f gpurun_out/$r.ncu-rep
done
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline.log 2>&1
timeout 120 python tools/tl_summary.py gpurun_out/timeline.json > gpurun_out/timeline_summary.txt 2>&1
rm -f gpurun_out/timeline.json
du -sh gpurun_out
echo done
