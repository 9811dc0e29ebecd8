import sys
sys.path.insert(0, 'tests')
from conftest import small_case
from test_gpu_parity import engine
c = small_case(sys.argv[1])
eng = engine(c["res"], c["origin"], c["kind"], c["phi"])
eng.set_reference(c["a"]); eng.set_query(c["b"])
print("evaluating", flush=True)
mi, st, hist, total = eng.evaluate(c["poses"][:1], histograms=True)
print("done", st, mi, flush=True)
