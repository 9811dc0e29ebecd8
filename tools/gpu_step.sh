mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2e_pytest.log
timeout 900 python -m pytest tests/test_gpu_headline_parity.py -x -q -k "c4 or c5" >> gpurun_out/r2e_pytest.log 2>&1; echo "pytest2 rc=$?" >> gpurun_out/r2e_pytest.log
VARIANTS="base prev" CONFIGS="c4 c2 c1" bash tools/ab_run.sh > gpurun_out/r2e_ab.txt 2>&1
