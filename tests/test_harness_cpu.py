"""Host-side logic of the harness (no GPU): the chain-survival configuration contract
(SPEC.md:395-401 ChainConfig invariants) and the first-failure index helper."""

import pytest
import torch


@pytest.fixture(scope="module")
def h():
    from paper_2510_03426_b200 import harness

    return harness


def test_chain_config_invariants(h):
    cfg = h.ChainConfig(d=8, T_max=100, backend="goom32", seed=3, trials=2)
    assert (cfg.d, cfg.T_max, cfg.trials) == (8, 100, 2)
    for bad in (dict(d=0, T_max=1, backend="real64"), dict(d=1, T_max=0, backend="real64"),
                dict(d=1, T_max=1, backend="real64", trials=0),
                dict(d=1, T_max=1, backend="float8")):
        with pytest.raises(ValueError):
            h.ChainConfig(**bad)


def test_first_failure_index(h):
    bad = torch.tensor([[False, False, True], [False, True, True], [False, False, False]])
    # columns: never fails -> T (3), fails from step 1, fails from step 0
    assert h._first_failure(bad).tolist() == [3, 1, 0]


def test_growth_rate_of_a_straight_line(h):
    dg = torch.zeros(101, 4)
    dg[:, 1] = torch.arange(101, dtype=torch.float32) * 0.5
    assert abs(h.growth_rate(dg) - 0.5) < 1e-6
