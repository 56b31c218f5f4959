#!/bin/bash
# full ncu capture of the three-pass 3D kernels (12-band shard driver)
cd "$(dirname "$0")/.."
O=gpurun_out
R=${1:-r2}
python tools/prof3d.py 192 > $O/plain3_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k3s_" -s 3 -c 3 \
    -o $O/split3d_$R python tools/prof3d.py 192 > $O/ncu_split3d_$R.log 2>&1
echo done
