# development: the scaling run's first pass with the per-element math stripped (libfmm_b200_exp.so,
# -DFMM_SCALE_EXP; results invalid past P0) against the product library, fused and unfused
L=paper_1507_00687_b200/libfmm_b200.so
cp $L /tmp/lib_prod.so
for v in prod exp; do
  if [ $v = exp ]; then cp paper_1507_00687_b200/libfmm_b200_exp.so $L; else cp /tmp/lib_prod.so $L; fi
  for f in 1 0; do echo "$v fuse=$f"; FMM_SCALE_FUSE=$f bash tools/gpu/scale_trace.sh; done
done
cp /tmp/lib_prod.so $L
