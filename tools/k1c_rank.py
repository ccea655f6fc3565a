"""One rank of the K1C (fused accumulate + all-reduce over CUDA-IPC peer memory) two-rank check, as its own
process so that compute-sanitizer can wrap each rank directly:

    compute-sanitizer --tool memcheck python tools/k1c_rank.py 0 PORT OUT &
    compute-sanitizer --tool memcheck python tools/k1c_rank.py 1 PORT OUT
    python tools/k1c_rank.py check OUT

Same workload as tests/test_dp_gpu.py::test_fused_peer_allreduce_two_ranks_one_gpu (2 ranks on cuda:0,
3 mini-batches of 2 x 12 samples as micro-batches of 4). ``check`` asserts both ranks hold identical weights.
"""
import os
import pickle
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class _FileQueue:
    def __init__(self, path):
        self.path = path

    def put(self, item):
        with open(self.path, "wb") as f:
            pickle.dump(item, f)


if __name__ == "__main__":
    if sys.argv[1] == "check":
        out = sys.argv[2]
        r0, r1 = (pickle.load(open(f"{out}.{r}.pkl", "rb")) for r in (0, 1))
        np.testing.assert_array_equal(r0[1], r1[1])
        np.testing.assert_array_equal(r0[3], r1[3])
        print("k1c two ranks: identical weights and reduced accumulators; losses", [o[0] for o in r0[2]])
    else:
        from tests.test_dp_gpu import _rank_peer
        rank, port, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
        _rank_peer(rank, 2, port, 12, 4, "exact_weighted", _FileQueue(f"{out}.{rank}.pkl"))
