# Session 4: ncu --set full of cfg5's HBM-bound kernels (k_combine_t, k_combine_all, k_expand4_rows7).
mkdir -p gpurun_out/s4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_combine_t|k_combine_all|k_expand4_rows7|k_transpose' --launch-skip 12 -c 12 -o gpurun_out/s4/cfg5_hbm python tools/cfg5_once.py > gpurun_out/s4/ncu_cfg5.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/s4/cfg5_hbm.ncu-rep > gpurun_out/s4/cfg5_hbm_summary.txt 2>&1; tail -5 gpurun_out/s4/cfg5_hbm_summary.txt
