for g in 1 2 4 8 16 32 64 128; do
  echo "group $g"
  TD_GEMM_GROUP=$g python tools/tuning/tune2.py 20 20 1 2>&1 | grep 16384
  TD_GEMM_GROUP=$g ncu --metrics dram__bytes_read.sum --clock-control none -k regex:dgemm_kernel -s 1 -c 1 python tools/tuning/prof2.py gemm 2>&1 | grep dram__
done
