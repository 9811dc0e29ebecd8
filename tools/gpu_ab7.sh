VARIANTS="base st3" CONFIGS="c4" bash tools/ab_run.sh 2>&1 | grep -v "^+"
for f in 1.3 1.6 2.0; do echo "capm $f"; VMI_CAPM_FACTOR=$f VARIANTS="base" CONFIGS="c4" bash tools/ab_run.sh 2>&1 | grep -v "^+"; done
VARIANTS="base st3" CONFIGS="c4" bash tools/ab_run.sh 2>&1 | grep -v "^+"
