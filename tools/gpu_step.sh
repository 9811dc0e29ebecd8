mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2af_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2af_pytest.log
timeout 900 python -m pytest tests/test_gpu_headline_parity.py -x -q -k "c4 or c2_batch" >> gpurun_out/r2af_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2af_pytest.log
AB="base nosat:VMI_SAT_MB=0" CONFIGS="c1 c2 c4 c3" bash tools/ab_env.sh > gpurun_out/r2af_ab.txt 2>&1
