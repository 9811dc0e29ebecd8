VARIANTS="base" CONFIGS="c2" bash tools/ab_run.sh 2>&1 | grep -v "^+"
echo "--- VMI_FORCE_F64 (double records)"
VMI_FORCE_F64=1 VARIANTS="base d4 d6" CONFIGS="c2" bash tools/ab_run.sh 2>&1 | grep -v "^+"
