import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The GPU tests exercise each top-k kernel path on small shapes: keep small calls on the fused
# tensor-core kernel (the product routes nq * ndb <= 2^25 to the CUDA-core kernels; that rule has its
# own test, test_topk_small_call_routing, which switches it back on).
os.environ.setdefault("BINSKETCH_TOPK_SMALL", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running statistical test")
