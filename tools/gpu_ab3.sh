set -x
VARIANTS="base pre19 base pre19" CONFIGS="c4 c2" bash tools/ab_run.sh 2>&1 | grep -v "^+"
for f in 2.0 1.7 3.0; do echo "cap factor $f"; VMI_CAP_FACTOR=$f VARIANTS="base" CONFIGS="c2" bash tools/ab_run.sh 2>&1 | grep -v "^+"; done
