# full GPU suite, smoke, N=1 bench (used for the per-change records)
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_g1.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_g1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_g1.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_g1.json 2> gpurun_out/bench_g1.err
