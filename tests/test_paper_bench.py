"""The paper's §5 kernel comparison (paper_1804_02221_b200/paper_bench.py): the
closed-form operation counts against the reference's CountReal instrumentation
(bench::count_ops, bench.hpp:160-192), and on the GPU the split-form and standard
volume kernels (csrc/kernels_bench.cu) against the reference's
kernels::split_volume_element / standard_volume_element (dg_rhs.hpp:23-117)."""
import numpy as np
import pytest

from oracle import ref
from paper_1804_02221_b200 import paper_bench
from tests.conftest import gpu_available
from tests.helpers import normwise


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("N", list(range(1, 16)))
def test_counts_match_reference_counter(N):
    assert paper_bench.counts(N, 3) == ref.count_ops(N, 3)


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("N", list(range(1, 16)))
def test_volume_kernels_match_reference(N):
    import torch
    K = 37
    n = K * (N + 1) ** 2
    rng = np.random.default_rng(N)
    h = rng.uniform(0.5, 2.0, n)
    h[rng.uniform(0, 1, n) < 0.05] = 0.0  # dry nodes: the velocity floor
    ins = [h, h * rng.uniform(-1, 1, n), h * rng.uniform(-1, 1, n),
           rng.uniform(0.3, 0.7, n), rng.uniform(-0.1, 0.1, n), rng.uniform(-0.1, 0.1, n),
           rng.uniform(0.3, 0.7, n)]
    dins = [torch.tensor(a, device="cuda") for a in ins]
    for kind in (0, 1):
        douts = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(3)]
        paper_bench.run_kernel(kind, N, K, dins, douts)
        torch.cuda.synchronize()
        got = [d.cpu().numpy() for d in douts]
        want = ref.volume_kernel(kind, N, K, ins)
        assert normwise(got, want) <= 1e-12, (kind, normwise(got, want))
