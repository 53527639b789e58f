# k_m4rm geometry sweep (each geometry its own process): 4096^3 and cfg4's shape.
for shape in "4096 4096 4096" "10000 7001 12345" "8192 8192 8192"; do
  for geom in "" "16,2" "16,4" "12,2" "12,4" "12,6" "8,2" "8,4" "8,8" "4,4" "4,3"; do
    echo "$shape geom=${geom:-model} $(GF2_M4RM_GEOM=$geom python tools/m4rm_geom.py $shape 2>&1 | tail -1 | cut -c1-200)"
  done
done
