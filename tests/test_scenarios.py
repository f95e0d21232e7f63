"""Scenario builders (CPU)."""
import numpy as np


def test_scenario_ic_matches_host_build():
    """The column-equilibrium IC spec reproduces the default host build
    (CPU; the device builder is checked against it in test_gpu_ic.py)."""
    from paper_1806_04960_b200.scenarios import build_scenario
    for name, res in (("wall-impact", (64, 36)), ("lake", (64, 32)), ("weir", (120, 40))):
        sc = build_scenario(name, res)
        lazy = build_scenario(name, res, host_state=False)
        assert lazy.q0 is None
        assert np.array_equal(lazy.ic.host_state(lazy.grid, lazy.params), sc.q0)
