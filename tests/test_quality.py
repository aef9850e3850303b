"""Eviction-quality metrics (eviction_loss.hpp) on device outputs, SURVEY §8(f) item 3."""
import numpy as np
import pytest
import torch

from paper_2407_11550_b200 import quality
from paper_2407_11550_b200._lib import InvalidArgument


def test_metric_definitions_match_reference_formulas():
    rng = np.random.default_rng(2)
    w = rng.random((3, 5, 40))
    keep = (rng.random((3, 5, 40)) < 0.3).astype(np.uint8)
    wt, kt = torch.as_tensor(w), torch.as_tensor(keep)
    # eviction_loss.hpp:64-78 / 44-61 restated per problem
    ret = np.array([sum(w[p, i, j] for i in range(5) for j in range(40) if keep[p, i, j]) for p in range(3)])
    ev = np.array([sum(w[p, i, j] for i in range(5) for j in range(40) if not keep[p, i, j]) for p in range(3)])
    assert np.allclose(quality.retained_mass(wt, kt).numpy(), ret, rtol=1e-13)
    assert np.allclose(quality.epsilon_bound(wt, kt, 1.5).numpy(), 3.0 * ev, rtol=1e-13)
    assert quality.l1_eviction_loss(torch.tensor([1.0, -2.0]), torch.tensor([0.5, 1.0])) == 3.5
    # a fully retained decision has zero bound (eviction_loss.hpp:44-46)
    assert float(quality.epsilon_bound(wt, torch.ones_like(kt), 2.0).abs().max()) == 0.0
    with pytest.raises(InvalidArgument):
        quality.epsilon_bound(wt, kt, -1.0)
    with pytest.raises(InvalidArgument):
        quality.l1_eviction_loss(torch.zeros(2), torch.zeros(3))


@pytest.mark.gpu
def test_adaptive_retains_more_mass_than_uniform(dev):
    """Algorithm 1's layer-wide top-B maximises retained mass before the safeguard; with the
    alpha = 0.2 blend it still retains at least as much as uniform allocation on planted heads
    (Theorem 3.3 / Fig. 3), and its decode output is closer to full attention."""
    from paper_2407_11550_b200.synthetic import planted_layer
    P, H, G, m, n_o, d = 6, 32, 8, 32, 8160, 128
    q, k, v = planted_layer(P, H, G, n_o, m, d, seed=17, dtype=torch.bfloat16, device=dev)
    r = quality.compare_allocations(q, k, v, 512 * G)
    ra, ru = r["retained_ada"].cpu().numpy(), r["retained_uniform"].cpu().numpy()
    assert np.all(ra >= ru * (1 - 1e-6)), (ra, ru)
    la, lu = r["l1_ada"].cpu().numpy(), r["l1_uniform"].cpu().numpy()
    assert (la <= lu).mean() >= 0.5, (la, lu)
