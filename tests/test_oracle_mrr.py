"""Pins of the oracle's LP MRR (Tables 2 and 6 report it; reading R-mrr: ties count
half) against closed forms and brute force over tie orders."""
import itertools

import numpy as np

import oracle


def test_mrr_hand_example():
    # pos 0.5; negatives 0.7 (higher), 0.5 (tie), 0.1 (lower) -> rank 2.5
    rr, m = oracle.lp_mrr(np.array([[0.5, 0.7, 0.5, 0.1]]))
    assert rr[0] == 1 / 2.5 and m == 0.4


def test_mrr_closed_forms():
    K = 7
    lower = np.concatenate([np.ones((3, 1)), np.zeros((3, K))], axis=1)
    higher = np.concatenate([np.zeros((3, 1)), np.ones((3, K))], axis=1)
    equal = np.ones((3, K + 1))
    assert oracle.lp_mrr(lower)[1] == 1.0
    assert np.isclose(oracle.lp_mrr(higher)[1], 1 / (K + 1))
    assert np.isclose(oracle.lp_mrr(equal)[1], 1 / (1 + K / 2))
    # MRR is the mean of the rows' reciprocal ranks
    rr, m = oracle.lp_mrr(np.concatenate([lower[:1], higher[:1]]))
    assert np.isclose(m, (1 + 1 / (K + 1)) / 2)


def test_mrr_rank_is_expected_rank_over_tie_orders():
    """Brute force: list the row in every order that sorts by descending score (ties in every
    permutation); the positive's mean 1-based position equals 1 / rr."""
    rng = np.random.default_rng(7)
    for _ in range(30):
        K = int(rng.integers(1, 6))
        row = rng.integers(0, 3, size=K + 1).astype(np.float64)     # small integers: many ties
        positions = []
        for perm in itertools.permutations(range(K + 1)):
            order = sorted(perm, key=lambda j: -row[j])             # stable: ties keep perm order
            positions.append(order.index(0) + 1)
        rr, _ = oracle.lp_mrr(row[None, :])
        assert np.isclose(1 / rr[0], np.mean(positions))


def test_mrr_rank_invariances():
    rng = np.random.default_rng(3)
    S = rng.normal(size=(50, 33))
    rr, m = oracle.lp_mrr(S)
    # a monotone transform of all scores keeps every rank; shuffling the negatives too
    rr2, _ = oracle.lp_mrr(2.0 * S + 1.0)
    perm = np.concatenate([[0], 1 + rng.permutation(32)])
    rr3, _ = oracle.lp_mrr(S[:, perm])
    assert np.array_equal(rr, rr2) and np.array_equal(rr, rr3)
    # without ties the rank is 1 + the number of higher negatives, in [1, K + 1]
    assert np.all((1 / rr >= 1) & (1 / rr <= 33))
    assert np.allclose(1 / rr, 1 + (S[:, 1:] > S[:, :1]).sum(axis=1))
