#!/bin/bash
# Classification kernels (tile classes + sub-unit masks) of the culled C5 plan
# per tuning variant (tools/build_variants.sh "cm1:-DGLR_XCLASSMINB=1" ...):
#   bash tools/classtime.sh cm1 cm2 u4 u8
for v in "$@"; do
  GLARE_B200_LIB=tools/variants/$v/libglare_b200.so ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/lc_$v.csv python tools/c5_culled_once.py > /dev/null 2>&1
  echo $v $(grep -E "sub_mask_kernel|tile_class_kernel" gpurun_out/lc_$v.csv | awk -F'","' '{gsub(/"/,"",$NF); s+=$NF} END {print s/1e6 " ms class total"}')
done
