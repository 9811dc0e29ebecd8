mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2t_pytest.log
AB="base noregroup:VMI_REGROUP=0" CONFIGS="c1v c1 c2" bash tools/ab_env.sh > gpurun_out/r2t_ab.txt 2>&1
