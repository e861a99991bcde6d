"""Seeded input generators (synthetic/): shapes, determinism and the recipes DESIGN.md §4 states."""
import numpy as np
import pytest

from synthetic import get, make_inputs, shard_range
from synthetic.configs import CONFIGS, CONFIG_INDEX


def test_every_config_has_a_seed_index():
    assert set(CONFIGS) == set(CONFIG_INDEX)
    assert len(set(CONFIG_INDEX.values())) == len(CONFIG_INDEX)


@pytest.mark.parametrize("name", ["c1", "img32", "img64"])
def test_deterministic_and_normalised(name):
    cfg = get(name)
    x1, y1, a1, b1 = make_inputs(cfg)
    x2, y2, a2, b2 = make_inputs(cfg)
    for u, v in ((x1, x2), (y1, y2), (a1, a2), (b1, b2)):
        assert np.array_equal(u, v)
    assert x1.shape == (cfg.n, cfg.d) and y1.shape == (cfg.m, cfg.d)
    assert abs(a1.sum() - 1) < 1e-13 and abs(b1.sum() - 1) < 1e-13
    assert (a1 > 0).all() and (b1 > 0).all()


def test_image_workloads_are_pixel_grids():
    """NEXT-1 image pairs: both measures live on the same K x K pixel-centre grid and carry two
    independent smooth gray-level fields (DOTmark stand-in)."""
    for K in (32, 64):
        x, y, a, b = make_inputs(get(f"img{K}"))
        assert np.array_equal(x, y)
        i = (np.arange(K) + 0.5) / K
        assert np.array_equal(np.unique(x[:, 0]), i) and np.array_equal(x[K + 3], [i[1], i[3]])
        assert not np.allclose(a, b)
        # smooth field: neighbouring pixels differ far less than the dynamic range
        A = a.reshape(K, K)
        assert np.abs(np.diff(A, axis=0)).max() < 0.5 * (A.max() - A.min())


def test_shards_cover_the_workload():
    cfg = get("img32")
    x, *_ = make_inputs(cfg)
    parts = [x[slice(*shard_range(cfg.n, r, 3))] for r in range(3)]
    assert np.array_equal(np.concatenate(parts), x)
