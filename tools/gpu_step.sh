mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_pair or align_batch" > gpurun_out/r2w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2w_pytest.log
VMI_NO_GROUP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_pair or align_batch" >> gpurun_out/r2w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2w_pytest.log
timeout 900 python -m pytest tests/test_gpu_headline_parity.py -x -q -k "c5" >> gpurun_out/r2w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2w_pytest.log
VMI_TRACE=1 timeout 1200 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/r2w_c5.json 2> gpurun_out/r2w_c5.err
