set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab2.log
VARIANTS="base" CONFIGS="c2 c1 c4 c2 c4" bash tools/ab_run.sh > gpurun_out/ab2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pose_fast -s 3 -c 1 -f -o gpurun_out/k1_c4_v17 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c4.log 2>&1
