#!/bin/bash
# Round profiling recipe (run under gpurun): plain bench, ncu launch list of the
# same bench command, and one full ncu capture of the dominant 2D / 3D kernels.
set -u
R=${1:-r1}
cd "$(dirname "$0")/.."
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$R.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k2_|k3_" -c 300 --csv \
    --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_$R.log 2>&1
python tools/prof2d.py denoise > gpurun_out/plain2_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k2_rows_fused|k2_cols_dec|k2_cols_rec|k2_cols_sum" -s 8 -c 4 \
    -o gpurun_out/full2d_$R python tools/prof2d.py denoise > gpurun_out/ncu_full2d_$R.log 2>&1
python bench.py --config 3d192 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench3d_$R.json 2> gpurun_out/bench3d_$R.err
echo done
