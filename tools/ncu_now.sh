cd $GRAFT_REPO_ROOT
O=gpurun_out
python tools/prof2d.py denoise > $O/plain2_r2a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k2_rows_fused|k2_cols_dec|k2_cols_rec|k2_cols_sum" -s 8 -c 4 \
    -o $O/full2d_r2a python tools/prof2d.py denoise > $O/ncu_full2d_r2a.log 2>&1
python tools/prof3d.py 192 > $O/plain3_r2a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k3_|k2_rows_fused" -s 11 -c 6 \
    -o $O/full3d_r2a python tools/prof3d.py 192 > $O/ncu_full3d_r2a.log 2>&1
echo done
