mkdir -p gpurun_out
V=v22
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$V.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$V.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$V.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$V.log
timeout 600 python bench.py > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$V.json 2> gpurun_out/bench_ref_$V.err
tail -3 gpurun_out/pytest_gpu_$V.log; cat gpurun_out/smoke_$V.log | tail -3; cat gpurun_out/bench_$V.json gpurun_out/bench_ref_$V.json
