mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_pair or align_batch" > gpurun_out/r2y_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2y_pytest.log
timeout 900 python -m pytest tests/test_gpu_headline_parity.py -x -q -k "c5" >> gpurun_out/r2y_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2y_pytest.log
timeout 1200 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/r2y_c5.json 2> gpurun_out/r2y_c5.err
