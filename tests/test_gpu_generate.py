"""Problems built on the device (csrc/generate_kernels.cu, C ABI
ssqa_problem_create_dense / ssqa_problem_create_gi): the quantized device
image must equal the one the host builders + ssqa_problem_create produce
(which the golden fixtures pin to the reference), and the fresh-instance
battery built this way must reproduce the reference's run_trials
(fresh_instance, bench.cpp:387-389) at the C3 size.
"""
import numpy as np
import pytest

import paper_2302_12454_b200 as sq

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def same_problem(a, b):
    ja, ha, oa = a.export()
    jb, hb, ob = b.export()
    assert a.info() == b.info()
    assert np.array_equal(ja, jb)
    assert np.array_equal(ha, hb)
    assert np.array_equal(bits(oa), bits(ob))


@pytest.mark.parametrize("n,kind", [(100, 0), (1000, 1), (2000, 0), (129, 1)])
def test_dense_generator_matches_host_builder(n, kind):
    same_problem(sq.Problem.generated_dense(n, kind, 7), sq.Problem(sq.dense_ising(n, kind, 7)))


@pytest.mark.parametrize("nn,seed,permute,c1,c2", [(10, 7, True, 1.0, 1.0),
                                                   (20, 3, False, 0.75, 0.75),
                                                   (7, 11, True, 0.5, 2.0),
                                                   (2, 5, True, 1.0, 1.0),
                                                   (13, 9, True, 1.25, 0.375)])
def test_gi_generator_matches_host_builder(nn, seed, permute, c1, c2):
    same_problem(sq.Problem.generated_gi(nn, [seed], 0.5, permute, c1, c2),
                 sq.Problem(sq.gi_ising(nn, 0.5, seed, permute, c1, c2)))


def test_gi_generator_many_matches_from_models():
    seeds = sq.trial_instance_seeds(1000, 24)
    models = [sq.gi_ising(10, 0.5, s, False, 0.75, 0.75) for s in seeds]
    same_problem(sq.Problem.generated_gi(10, seeds, 0.5, False, 0.75, 0.75),
                 sq.Problem.from_models(models))


def test_gi_generator_rejects_non_dyadic_penalty():
    with pytest.raises(sq.SsqaInvalidArgument):
        sq.Problem.generated_gi(6, [1], 0.5, True, 0.7, 0.3)


def test_fresh_battery_at_c3_size_matches_reference(golden):
    """run_trials with a fresh GI instance per trial at n = 50 (N = 2500), the
    whole 1024-trial battery as one device batch of device-built instances;
    the trials the reference ran (scripts/make_golden.py: oracle/_ref
    run_trials(fresh_instance), 16 trials at sc = 5000) must match."""
    ref = golden("trials_large")["c3_fresh_gi50"]
    outs, p_s, _, _ = sq.run_trials_fresh(50, sq.SsqaParams(r=20), 1024, 100000, 1000,
                                          permute=True, c1=1.0, c2=1.0)
    k = len(ref["seed"])
    assert [o.seed for o in outs[:k]] == [int(x) for x in ref["seed"]]
    assert [int(o.reached_target) for o in outs[:k]] == [int(x) for x in ref["reached"]]
    assert [o.first_hit_cycle for o in outs[:k]] == [int(x) for x in ref["first_hit"]]
    assert np.array_equal(bits([o.best_energy for o in outs[:k]]), bits(ref["best_energy"]))
