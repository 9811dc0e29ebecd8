# A/B: 9-deep cp.async ring (3 push groups in flight), +1024-entry walk ring
VARIANTS="base s9 s9w1024" CONFIGS="c2 c1" bash tools/ab_run.sh 2>&1 | grep -v "^+"
VARIANTS="base s9 s9w1024" CONFIGS="c2" bash tools/ab_run.sh 2>&1 | grep -v "^+"
