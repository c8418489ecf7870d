mkdir -p gpurun_out
P="python scripts/prof_pull.py --config c2 --launches 6"
for L in build_alt/libprgpu_head.so paper_2108_02997_b200/libprgpu.so; do
  tag=$(basename $L .so)
  PRGPU_LIB=$L timeout 200 $P > gpurun_out/p_$tag.log 2>&1 && PRGPU_LIB=$L timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/w_$tag $P > gpurun_out/n_$tag.log 2>&1; echo "$tag rc=$?"
done
