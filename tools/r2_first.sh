mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2a_gpus.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2a_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r2a_bench_rmat20.json 2> gpurun_out/r2a_bench_rmat20.err; echo bench rc=$?; cat gpurun_out/r2a_bench_rmat20.json | head -c 600
