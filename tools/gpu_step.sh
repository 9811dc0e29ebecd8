mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s_pytest.log
VARIANTS="base prev" CONFIGS="c1" bash tools/ab_run.sh > gpurun_out/r2s_ab.txt 2>&1
