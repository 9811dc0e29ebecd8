mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2ah_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ah_pytest.log
timeout 900 python -m pytest tests/test_gpu_headline_parity.py -x -q -k "c4" >> gpurun_out/r2ah_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ah_pytest.log
VARIANTS="base prev base prev" CONFIGS="c4" bash tools/ab_run.sh > gpurun_out/r2ah_ab.txt 2>&1
