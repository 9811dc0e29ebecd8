mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "not c5_pairs" > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 600 python bench.py > gpurun_out/r2a_bench_c2.json 2> gpurun_out/r2a_bench_c2.err
AB="base cta256:VMI_CTA_THREADS=256,VMI_SINGLE_MAXLOAD=0.9" CONFIGS="c2 c3 c1 c4" bash tools/ab_env.sh > gpurun_out/r2a_ab.txt 2>&1
