import sys, time
sys.path.insert(0, 'tests')
import numpy as np
from conftest import small_case
from test_gpu_parity import engine
tag = sys.argv[1]
c = small_case(tag)
eng = engine(c["res"], c["origin"], c["kind"], c["phi"])
eng.set_reference(c["a"]); eng.set_query(c["b"])
print("f32", eng.ctx.__dict__.get('is_f32', '?'), flush=True)
for k in range(c["poses"].shape[0]):
    t = time.time()
    mi, st, hist, total = eng.evaluate(c["poses"][k:k+1], histograms=True)
    print(k, st, mi, np.array_equal(hist[0], c["hist"][k]), round(time.time()-t, 3), flush=True)
