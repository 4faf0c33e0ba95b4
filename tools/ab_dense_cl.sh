# K3c cluster size A/B on the cfg3 batch (OTK_DENSE_CL forces the size; default = the planner's choice)
for rep in 1 2; do
for cl in "" 5 6 7 8; do
  echo "== CL=${cl:-auto}"
  OTK_DENSE_CL=$cl python tools/ab_dense.py paper_2201_12324_b200/libotk_sm100.so 2>&1 | grep median
done
done
