mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2ac_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ac_pytest.log
VARIANTS="base w128 s9 base" CONFIGS="c4 c2 c3" bash tools/ab_run.sh > gpurun_out/r2ac_ab.txt 2>&1
