# Session 4: k_combine_t with STG.256 stores (cfg5 timeline), per-rank compute on process grids.
mkdir -p gpurun_out/s4
python -m pytest tests/test_gpu_parity.py -x -q -k "cfg5 or deep or depth or strassen" > gpurun_out/s4/b_tests.log 2>&1; tail -2 gpurun_out/s4/b_tests.log
python tools/timeline.py --size 65536 --addmul --summary --reps 2 > gpurun_out/s4/b_timeline_cfg5.txt 2>&1; cat gpurun_out/s4/b_timeline_cfg5.txt
python tools/grid_estimate.py 16384 2 > gpurun_out/s4/b_grid_cfg3.txt 2>&1; cat gpurun_out/s4/b_grid_cfg3.txt
python tools/grid_estimate.py 65536 2 > gpurun_out/s4/b_grid_cfg5.txt 2>&1; cat gpurun_out/s4/b_grid_cfg5.txt
