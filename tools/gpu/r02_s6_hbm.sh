# Round-2 session 6: ncu --set full of the HBM-bound kernels of one cfg5 addmul
# (second call of tools/cfg5_once.py: the first warms the workspace pool).
mkdir -p gpurun_out/s6
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_combine_t --launch-skip 1 -c 1 -o gpurun_out/s6/combine_t python tools/cfg5_once.py > gpurun_out/s6/ncu_ct.log 2>&1; echo "ncu combine_t rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:k_combine_all --launch-skip 5 -c 5 -o gpurun_out/s6/combine_all python tools/cfg5_once.py > gpurun_out/s6/ncu_ca.log 2>&1; echo "ncu combine_all rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:k_expand4_rows7 --launch-skip 6 -c 2 -o gpurun_out/s6/expand python tools/cfg5_once.py > gpurun_out/s6/ncu_ex.log 2>&1; echo "ncu expand rc=$?"
