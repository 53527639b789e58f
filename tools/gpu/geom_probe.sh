mkdir -p gpurun_out
for shp in "1024 1024 1024" "1000 1100 1300" "2048 2048 2048"; do
  for gm in 16,1 16,8 8,8 4,8 4,4 2,4 2,8 model; do
    if [ $gm = model ]; then timeout 120 python tools/m4rm_geom.py $shp 2>&1 | tail -1;
    else GF2_M4RM_GEOM=$gm timeout 120 python tools/m4rm_geom.py $shp 2>&1 | tail -1; fi
  done
done
for shp in "10000 7001 12345" "4096 4096 4096" "16384 16384 16384"; do timeout 300 python tools/m4rm_geom.py $shp 2>&1 | tail -1; done
