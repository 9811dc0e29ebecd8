mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "occupancy or kitti or hdl or small or c1 or fast_path" > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 600 python -m pytest tests/test_gpu_headline_parity.py -x -q -k "c4" >> gpurun_out/r2b_pytest.log 2>&1; echo "pytest2 rc=$?" >> gpurun_out/r2b_pytest.log
AB="base noocc:VMI_NO_OCC=1" CONFIGS="c4" bash tools/ab_env.sh > gpurun_out/r2b_ab.txt 2>&1
