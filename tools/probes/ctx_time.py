"""Context creation (upload + transpose) and first-evaluation (rank build) times."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_1801_03039_b200 as eb
from golden_io import trace
for name in sys.argv[1:] or ["c4", "c5"]:
    t = trace(name)
    a = time.perf_counter(); v = t.matrix(); b = time.perf_counter()
    eb.device_count()
    c = time.perf_counter(); ev = eb.Evaluator(v); d = time.perf_counter()
    off, cols, _, _ = t.batches[0]
    pop = eb.CbfPopulation(off, cols)
    ev.evaluate_population(pop, eb.FitnessParams(t.sigma), t.eps); e = time.perf_counter()
    ev.evaluate_population(pop, eb.FitnessParams(t.sigma), t.eps); f = time.perf_counter()
    print(f"{name}: generate {b-a:.3f}s  ctx_create {d-c:.3f}s ({v.nbytes/1e9:.2f} GB)  first_eval {e-d:.3f}s  second {1e6*(f-e):.0f}us", flush=True)
    ev.close()
