set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/a_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/a_ref.json 2> gpurun_out/a_ref.err
timeout 600 python bench.py --sharded --no-cpu-baseline > gpurun_out/a_sharded.json 2> gpurun_out/a_sharded.err
tail -3 gpurun_out/a_pytest.log; cat gpurun_out/a_bench.json gpurun_out/a_ref.json gpurun_out/a_sharded.json
