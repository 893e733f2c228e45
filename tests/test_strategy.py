"""Pivot strategies: byte-equality with the reference tables, plus the
reference's own structural tests (pkg/tests/test_strategy.py)."""

import hashlib
import itertools

import pytest

from paper_1401_2720_b200 import strategy as S


def _sha(s):
    return hashlib.sha256(S.dump_strategy(s).encode()).hexdigest()


def test_all_tables_match_reference_digests(strategies_golden):
    bad = []
    for key, want in strategies_golden["hash"].items():
        parts = key.split(":")
        if parts[0] == "expand":
            kind, n = parts[1], int(parts[2])
            got = _sha(S.expand_pstrategy(S.closest_pstrategy(kind, n), kind))
        else:
            kind, n = parts[0], int(parts[1])
            try:
                st = S.make_strategy(kind, n)
            except S.StrategyError as exc:
                got = "error:" + type(exc).__name__
            else:
                got = _sha(st)
                assert st.kind == strategies_golden["kindtag"][key], key
        if got != want:
            bad.append(key)
    assert not bad, bad


def test_small_tables_text_equal(strategies_golden):
    for key, txt in strategies_golden["text"].items():
        kind, n = key.split(":")
        assert S.dump_strategy(S.make_strategy(kind, int(n))) == txt, key


def test_row4_exact():
    # reference tests/test_strategy.py:23 (R4)
    r4 = S.closest_pstrategy("row", 4)
    assert r4.steps == (((1, 2), (3, 4)), ((1, 3), (2, 4)), ((1, 4), (2, 3)))


@pytest.mark.parametrize("n", [4, 6])
def test_closest_is_bruteforce_minimum(n):
    # SPEC acceptance 1: lexicographic minimum over all p-strategies
    for kind, ref in (("row", S.row_cyclic(n)), ("col", S.column_cyclic(n))):
        pairs = ref.pairs
        idx = ref.index_of()
        matchings = []
        verts = list(range(1, n + 1))

        def perfect(rem):
            if not rem:
                yield ()
                return
            a = rem[0]
            for b in rem[1:]:
                rest = [x for x in rem if x not in (a, b)]
                for m in perfect(rest):
                    yield ((a, b),) + m

        for m in perfect(verts):
            matchings.append(tuple(sorted(m, key=lambda pq: idx[pq])))
        best = None
        for combo in itertools.permutations(matchings, n - 1):
            flat = [pq for st in combo for pq in st]
            if len(set(flat)) != len(pairs):
                continue
            key = [idx[pq] for pq in flat]
            if best is None or key < best:
                best = key
        got = [idx[pq] for pq in S.closest_pstrategy(kind, n).flattened()]
        assert got == best


@pytest.mark.parametrize("n", [2, 4, 6, 8, 10, 12, 14, 16, 20, 24, 28, 32])
def test_lemma_3_2_first_step(n):
    for kind in ("row", "col"):
        st = S.make_strategy(kind, n)
        assert st.steps[0] == tuple((2 * k - 1, 2 * k) for k in range(1, n // 2 + 1))


@pytest.mark.parametrize("n", [4, 6, 8])
def test_duplication(n):
    for kind in ("row", "col"):
        assert (S.expand_pstrategy(S.closest_pstrategy(kind, n), kind).steps
                == S.closest_pstrategy(kind, 2 * n).steps)


@pytest.mark.parametrize("n", [4, 8, 16])
def test_step_equivalence_powers_of_two(n):
    assert S.step_equivalent(S.make_strategy("row", n), S.make_strategy("col", n))


@pytest.mark.parametrize("kind", ["row", "col", "rrow", "rcol", "bl", "mm"])
@pytest.mark.parametrize("n", [2, 8, 12, 24, 32, 64, 512])
def test_validity(kind, n):
    assert S.validate_pstrategy(S.make_strategy(kind, n)) == []


def test_reverse_involution_and_kind():
    st = S.make_strategy("row", 16)
    rv = S.reverse_pstrategy(st)
    assert rv.kind == "reversed-row"
    assert S.reverse_pstrategy(rv).steps == st.steps


def test_dump_parse_round_trip():
    st = S.make_strategy("rrow", 32)
    assert S.parse_strategy(S.dump_strategy(st)).steps == st.steps


def test_errors():
    with pytest.raises(S.StrategyError):
        S.make_strategy("row", 7)
    with pytest.raises(S.StrategyError):
        S.make_strategy("nope", 8)
    with pytest.raises(S.SearchBudgetExceeded):
        S.closest_pstrategy("row", 18)
    with pytest.raises(S.StrategyError):
        S.parse_strategy("4 3 2\n1:2 3:4\n")
    bad = S.PStrategy(4, (((1, 2), (3, 4)), ((1, 2), (3, 4)), ((1, 4), (2, 3))))
    assert S.validate_pstrategy(bad)
    with pytest.raises(S.StrategyError):
        S.reverse_pstrategy(bad)


def test_as_table_zero_based():
    tab = S.as_table(S.make_strategy("mm", 8))
    assert tab.shape == (7, 4, 2) and tab.dtype.name == "int32"
    assert tab.min() == 0 and tab.max() == 7
