"""Device-level photon partitioning (host C++ in libvoxmc_b200.so) vs the
reference (golden fixture + live oracle/_ref): test_scheduler.cpp:42-138,
acceptance.cpp criteria 6-8."""
import random

import pytest

import paper_1711_03244_b200 as v


def profs(ps):
    return [v.DeviceProfile(cores=c, a=a, t0=t0) for c, a, t0 in ps]


def test_golden_partitions(golden):
    for rec in golden["partitions"]:
        d = profs(rec["profiles"])
        for s in (1, 2, 3):
            assert v.make_partition(rec["total"], d, v.Strategy(s)).counts == rec[f"s{s}"]


def test_s1_examples():
    assert v.partition_s1(300, profs([(1, 1, 0), (2, 1, 0)])).counts == [100, 200]
    q = v.partition_s1(10, profs([(1, 1, 0)] * 3))
    assert q.counts == [4, 3, 3] and q.total() == 10  # lower-index tie break


def test_live_reference_random(ref):
    rnd = random.Random(3)
    for _ in range(150):
        k = rnd.randint(1, 6)
        ps = [(rnd.randint(1, 32), rnd.uniform(1e-5, 1e-2), rnd.uniform(0, 100)) for _ in range(k)]
        total = rnd.randint(0, 10**7)
        for s in (1, 2, 3):
            got = v.make_partition(total, profs(ps), v.Strategy(s)).counts
            want, span = ref.partition(s, total, ps)
            assert got == want
            assert sum(got) == total
            assert v.model_makespan(v.Partition(got), profs(ps)) == pytest.approx(span, rel=1e-12)


def test_s3_optimal_vs_brute_force(ref):
    rnd = random.Random(5)
    for _ in range(60):
        k = rnd.randint(2, 4)
        ps = [(1, rnd.uniform(0.5, 3.0), rnd.uniform(0, 20)) for _ in range(k)]
        total = rnd.randint(10, 400)
        p = v.partition_s3(total, profs(ps))
        _, best = ref.brute_force(total, ps)
        assert v.model_makespan(p, profs(ps)) == pytest.approx(best, rel=1e-9, abs=1e-9)


def test_strategy_ordering_paper_instance():
    """acceptance.cpp criterion 7: t0 = paper overheads, S3 <= S2 < S1."""
    d = profs([(28, 1.0e-4, 53.0), (22, 1.2e-4, 63.0), (64, 2.4e-4, 631.0), (36, 3.0e-4, 652.0)])
    total = 10**8 // 4
    m = {s: v.model_makespan(v.make_partition(total, d, s), d) for s in v.Strategy}
    assert m[v.Strategy.S3] <= m[v.Strategy.S2] < m[v.Strategy.S1]


def test_partition_errors():
    with pytest.raises(v.ValidationError):
        v.make_partition(10, [], v.Strategy.S1)
    with pytest.raises(v.ValidationError):
        v.partition_s2(10, profs([(1, 0.0, 0.0)]))
    with pytest.raises(v.ValidationError):
        v.partition_s1(10, profs([(0, 1.0, 0.0)]))
    assert v.thread_count_heuristic(12, 64) == 768
    with pytest.raises(v.ValidationError):
        v.thread_count_heuristic(0, 1)


def test_simulated_calibration():
    """scheduler.cpp:360-393 for simulated devices (exact model, jittered, flat)."""
    st = v.baseline_setup("b1", photons=1000)
    d = v.DeviceProfile(name="sim", a=0.002, t0=10.0, kind=v.DeviceKind.Simulated)
    cal = v.calibrate(d, 1000, 5000, st.scene, st.config)
    assert cal.a == pytest.approx(0.002) and cal.t0 == pytest.approx(10.0)
    d.jitter_sigma = 0.01
    cal = v.calibrate(d, 100_000, 500_000, st.scene, st.config, noise_seed=4)
    assert cal.a == pytest.approx(0.002, rel=0.1)
    flat = v.DeviceProfile(name="weird", a=0.0, t0=100.0, kind=v.DeviceKind.Simulated)
    with pytest.raises(v.NonPositiveSlope):
        v.calibrate(flat, 1000, 2000, st.scene, st.config)


def test_live_reference_ties_and_identical_devices(ref):
    """Identical and commensurate devices make many optimal S3 allocations tie;
    the split must still be the reference's, device for device (which device
    gets a tied unit depends on the FMA-rounded finish times a*n + t0)."""
    rnd = random.Random(9)
    cases = []
    for k in (1, 2, 3, 4, 8, 16, 17):
        for total in (0, 1, 2, 5, 7, 1000, 10**9 + 7):
            cases += [([(1, 1e-6, 0.1)] * k, total), ([(1, 1e-6, 0.0)] * k, total),
                      ([(1, 2e-6, 0.0), (1, 1e-6, 0.0)] * (k // 2 or 1), total),
                      ([(1, 1e-3, 5.0), (2, 1e-3, 0.0), (1, 1e-3, 5.0)] * (k // 3 or 1), total)]
    for _ in range(300):
        k = rnd.randint(1, 16)
        ps = [(rnd.randint(1, 64), rnd.choice([1e-6, 2e-6, 0.5, 0.25, rnd.uniform(1e-7, 1e-3)]),
               rnd.choice([0.0, 0.1, 1.0, rnd.uniform(0, 50)])) for _ in range(k)]
        cases.append((ps, rnd.choice([rnd.randint(0, 10**9), rnd.randint(0, 100)])))
    for ps, total in cases:
        for s in (1, 2, 3):
            want, _ = ref.partition(s, total, ps)
            if sum(want) != total:
                continue  # the reference's numerical corner, see the next test
            assert v.make_partition(total, profs(ps), v.Strategy(s)).counts == want, (s, total, ps)


def test_s3_covers_total_where_the_reference_returns_zeros(ref):
    """One device, 1e9 photons: the reference's bisection capacities
    floor((T - t0)/a + 1e-9) fall one photon short at its upper bound, so its
    S3 returns an all-zero split (scheduler.cpp:126-131,160). The B200 split
    gives the device every photon (the only valid split)."""
    want, _ = ref.partition(3, 10**9, [(1, 1e-6, 0.1)])
    assert want == [0]
    assert v.partition_s3(10**9, profs([(1, 1e-6, 0.1)])).counts == [10**9]
