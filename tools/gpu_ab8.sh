# A/B: two 256-thread CTAs per SM (epilogue/point-pass overlap) vs one 512-thread CTA
nvidia-smi --query-gpu=name,clocks.sm --format=csv
for v in c2x256 c2x256s3; do
  VMI_LIB=variants/$v/libvmi.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not thread_configurations" 2>&1 | tail -2
done
VARIANTS="base c2x256 c2x256s3" CONFIGS="c2 c1" bash tools/ab_run.sh 2>&1 | grep -v "^+"
VARIANTS="base c2x256" CONFIGS="c2" bash tools/ab_run.sh 2>&1 | grep -v "^+"
