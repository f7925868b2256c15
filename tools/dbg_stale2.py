import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2008_10596_b200 import engine as eng
import test_gpu_parity as T
L = eng.lib()
for seed in (1, 2, 3):
    try:
        T.test_random_mixed_paths_agree(eng, seed)
        print("seed", seed, "ok; pending error", L.crac_peek_cuda_error(), flush=True)
    except Exception as e:
        import traceback; traceback.print_exc()
        print("seed", seed, "FAILED", e, flush=True)
