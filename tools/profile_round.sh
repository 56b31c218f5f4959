#!/bin/bash
# Round profiling recipe (run under gpurun, one GPU): plain benches, ncu launch
# lists of the same bench commands, and one full ncu capture each of the
# dominant 2D / 3D kernels. Summarise afterwards with tools/ncu_summary.py.
set -u
R=${1:-r2}
cd "$(dirname "$0")/.."
O=gpurun_out
python bench.py --steps 50 --warmup 3 > $O/bench_$R.json 2> $O/bench_$R.err
python bench.py --config 3d128 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench3d128_$R.json 2> $O/bench3d128_$R.err
python bench.py --config 2d1024x64 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench1024_$R.json 2> $O/bench1024_$R.err
python bench.py --config 3d192sl1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench3dsl1_$R.json 2> $O/bench3dsl1_$R.err
python bench.py --config 3d256 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench3d256_$R.json 2> $O/bench3d256_$R.err
python bench.py --config 2d512_nostack --no-3d --steps 100 --warmup 3 --no-cpu-baseline > $O/benchnostack_$R.json 2> $O/benchnostack_$R.err
python bench.py --impl reference --steps 10 --warmup 1 > $O/bench_ref_$R.json 2> $O/bench_ref_$R.err
# launch lists (the bench commands that just exited 0, under ncu)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k2_|k3" -c 300 --csv \
    --log-file $O/launches_$R.csv python bench.py --no-3d --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch_$R.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k2_|k3" -c 300 --csv \
    --log-file $O/launches3d_$R.csv python bench.py --config 3d192 --steps 1 --warmup 1 --no-cpu-baseline \
    > $O/ncu_launch3d_$R.log 2>&1
# full captures of the dominant kernels (single-frame / 12-band drivers)
python tools/prof2d.py denoise > $O/plain2_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k2_rows_fused|k2_cols_dec|k2_cols_rec|k2_cols_sum" -s 8 -c 4 \
    -o $O/full2d_$R python tools/prof2d.py denoise > $O/ncu_full2d_$R.log 2>&1
python tools/prof3d.py 192 > $O/plain3_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k3g_|k3s_" -s 3 -c 3 \
    -o $O/full3d_$R python tools/prof3d.py 192 > $O/ncu_full3d_$R.log 2>&1
echo done
