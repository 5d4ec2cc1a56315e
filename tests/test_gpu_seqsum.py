"""deterministic_sum (parallel.hpp:50-54) on the device, bit for bit: the
reference's left-to-right sum (numpy's cumsum accumulates in the same order),
including ties to even at binade steps, terms that jump binades, zeros,
denormals, huge dynamic range and (ordered fallback) negative terms — and
average_edge_length / t = m h^2 now equal the reference's bits."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def seq(x):
    return float(np.cumsum(np.asarray(x, np.float64))[-1]) if len(x) else 0.0


@pytest.mark.parametrize("n", [1, 7, 4096, 4097, 5000, 100_003, 3_000_000])
def test_uniform_and_lognormal(gpu, n):
    g = gpu.geoheat
    rng = np.random.RandomState(n)
    for x in (rng.uniform(0, 1, n), np.exp(rng.normal(0, 6, n)), rng.uniform(0, 1e-3, n) * (rng.uniform(size=n) > 0.3)):
        assert g.deterministic_sum(x) == seq(x)


def test_ties_and_binade_jumps(gpu):
    g = gpu.geoheat
    rng = np.random.RandomState(7)
    n = 200_000
    # halves and quarters on a large running sum: exact ties at u = 1, 2, 4, ...
    x = rng.choice([0.5, 1.5, 0.25, 2.5, 1.0, 3.0], size=n)
    x[5000] = 2.0 ** 53  # a term far above the running sum (binade jump)
    x[100_000] = 2.0 ** 60
    assert g.deterministic_sum(x) == seq(x)
    y = np.concatenate([[2.0 ** 52], rng.choice([0.5, 1.0, 1.5], size=n)])
    assert g.deterministic_sum(y) == seq(y)
    # denormals and zeros
    z = np.concatenate([np.zeros(5000), rng.uniform(0, 1, 5000) * 5e-324 * 1e3, rng.uniform(0, 1e-300, 10_000)])
    assert g.deterministic_sum(z) == seq(z)


def test_prefix_saturation_and_mixed_scales(gpu):
    """Terms just below the first binade's top make that binade's integer
    prefix pass 2^63 (saturated, must stay monotone); mixed scales force
    many binade changes."""
    g = gpu.geoheat
    x = np.concatenate([np.ones(4096), np.full(300_000, 4095.9)])
    assert g.deterministic_sum(x) == seq(x)
    rng = np.random.RandomState(11)
    y = rng.uniform(0, 1, 500_000) * 10.0 ** rng.randint(-8, 8, 500_000)
    assert g.deterministic_sum(y) == seq(y)
    z = np.concatenate([np.full(4096, 1e-12), rng.uniform(0, 1, 1_000_000)])
    assert g.deterministic_sum(z) == seq(z)


def test_many_windows(gpu):
    """Terms spanning hundreds of binades (the running sum climbs through
    several 48-binade windows), tiny leading terms, denormal sums."""
    g = gpu.geoheat
    rng = np.random.RandomState(5)
    x = 10.0 ** rng.uniform(-300, 0, 400_000)
    assert g.deterministic_sum(x) == seq(x)
    y = np.concatenate([np.full(100_000, 1e-310), 10.0 ** np.linspace(-300, 300, 200_000)])
    assert g.deterministic_sum(y) == seq(y)
    z = np.sort(10.0 ** rng.uniform(-250, 250, 300_000))  # ascending: a new window every few segments
    assert g.deterministic_sum(z) == seq(z)


def test_negative_terms_take_the_ordered_path(gpu):
    g = gpu.geoheat
    rng = np.random.RandomState(3)
    x = rng.normal(0, 1, 50_000)
    assert g.deterministic_sum(x) == seq(x)
    assert g.deterministic_sum(np.array([])) == 0.0


@pytest.mark.parametrize("config,scale", [(1, 1), (2, 1), (3, 2), (4, 16)])
def test_average_edge_length_bitwise(gpu, port_oracle, config, scale):
    from paper_1812_06060_b200 import meshgen
    g = gpu.geoheat
    w = meshgen.config(config, scale=scale)
    mesh = g.build_mesh(w.positions, w.faces)
    om = port_oracle.build_mesh(w.positions, w.faces)
    assert g.average_edge_length(mesh) == om.average_edge_length()
    assert g.diffusion_time(mesh, 1.0) == om.diffusion_time(1.0)


def _same(a, b):
    return np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64) or (np.isnan(a) and np.isnan(b))


def test_batched_sums_every_family(gpu):
    """deterministic_sums (one device block per sum, the E1-group engine):
    every family above as rows of one batch — ties, binade jumps, denormals,
    saturating prefixes, hundreds of binades, zeros, negatives, inf and NaN."""
    g = gpu.geoheat
    rng = np.random.RandomState(21)
    n = 300_001
    rows = [
        rng.uniform(0, 1, n),
        np.exp(rng.normal(0, 6, n)),
        rng.uniform(0, 1e-3, n) * (rng.uniform(size=n) > 0.3),
        rng.choice([0.5, 1.5, 0.25, 2.5, 1.0, 3.0], size=n),
        np.concatenate([[2.0 ** 52], rng.choice([0.5, 1.0, 1.5], size=n - 1)]),
        np.concatenate([np.zeros(5000), rng.uniform(0, 1, 5000) * 5e-324 * 1e3, rng.uniform(0, 1e-300, n - 10000)]),
        np.concatenate([np.ones(4096), np.full(n - 4096, 4095.9)]),
        rng.uniform(0, 1, n) * 10.0 ** rng.randint(-8, 8, n),
        10.0 ** rng.uniform(-300, 0, n),
        np.concatenate([np.full(100_000, 1e-310), 10.0 ** np.linspace(-300, 300, n - 100_000)]),
        np.sort(10.0 ** rng.uniform(-250, 250, n)),
        rng.normal(0, 1, n),
        np.zeros(n),
        np.full(n, 5e-324),
        np.concatenate([rng.uniform(0, 1, 1000), [np.inf], rng.uniform(0, 1, n - 1001)]),
        np.concatenate([rng.uniform(0, 1, 1000), [np.nan], rng.uniform(0, 1, n - 1001)]),
        np.concatenate([rng.uniform(0, 1, 1000), [np.inf], rng.uniform(0, 1, 1000), [np.nan], np.ones(n - 2002)]),
        np.concatenate([[1e300] * 10, [1.7e308] * 3, rng.uniform(0, 1, n - 13)]),  # overflow to inf
        np.concatenate([rng.uniform(0, 1, n // 2), -rng.uniform(0, 1, n - n // 2)]),  # goes negative
    ]
    x = np.stack(rows)
    x[3, 5000] = 2.0 ** 53
    x[3, 100_000] = 2.0 ** 60
    got = g.deterministic_sums(x)
    for i, r in enumerate(x):
        assert _same(got[i], seq(r)), (i, got[i], seq(r))


@pytest.mark.parametrize("n", [1, 2, 4095, 4096, 4097, 8191, 12_289])
def test_batched_sums_ragged_tiles(gpu, n):
    """Lengths around the 4096-term tile, many rows of adversarial halves."""
    g = gpu.geoheat
    rng = np.random.RandomState(n)
    x = rng.choice([0.5, 1.5, 2.0 ** -53, 2.0 ** -54, 3.0 * 2.0 ** -54, 1.0], size=(37, n))
    x[:, 0] = 2.0 ** rng.randint(-60, 60, 37)
    got = g.deterministic_sums(x)
    for i, r in enumerate(x):
        assert _same(got[i], seq(r)), (i, got[i], seq(r))
    assert g.deterministic_sums(np.zeros((3, 0))).tolist() == [0.0, 0.0, 0.0]
