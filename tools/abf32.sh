# A/B the fp32-mode 3D path across prebuilt library variants (paper_1402_5670_b200/libab_<v>.so)
for v in ${VARIANTS:-A}; do
  echo "$v $(SLB_LIB=$PWD/paper_1402_5670_b200/libab_$v.so python tools/f32_3d.py 10)"
done
