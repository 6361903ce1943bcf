"""butterfly-schedule module: SPEC.md:178-265 examples and properties, for the
native schedule (libbflybfs, host-only) and the oracle restatement."""

import pytest

from oracle import schedule as osched
from paper_2103_13577_b200 import schedule as S


def test_paper_examples_fig1_fig2():
    # SPEC.md:199-201
    assert [r[0] for r in S.make_schedule(16, 1)] == [(1,), (2,), (4,), (8,)]
    s = S.make_schedule(16, 4)
    assert s[0][0] == (1, 2, 3)
    assert s[1][0] == (4, 8, 12)


def test_nine_node_bottleneck():
    # SPEC.md:201, acceptance 5
    last = S.make_schedule(9, 1)[-1]
    assert [last[g] for g in range(8)] == [(8,)] * 8
    assert sum(1 for srcs in last for s in srcs if s == 8) == 8


def test_num_rounds():
    # SPEC.md:208-210, acceptance 3
    assert S.num_rounds(16, 1) == 4
    assert S.num_rounds(16, 4) == 2
    assert S.num_rounds(9, 1) == 4
    assert S.num_rounds(1, 1) == 0


def test_message_counts():
    # SPEC.md:217-219,226-228, acceptance 2
    assert S.message_count_paper(16, 1) == 64
    assert S.message_count_paper(16, 4) == 128
    assert S.message_count_paper(16, 16) == 256
    assert S.message_count_remote(S.make_schedule(16, 1)) == 64
    assert S.message_count_remote(S.make_schedule(16, 4)) == 96
    assert S.message_count_remote(S.make_schedule(1, 1)) == 0
    assert S.message_count_remote(S.all_to_all_schedule(16)) == 240


def test_buffer_bound():
    # SPEC.md:235-237, acceptance 4
    assert S.buffer_bound(1000, 4) / S.buffer_bound(1000, 1) == 4
    assert S.buffer_bound(0, 3) == 0
    assert S.buffer_bound(10**6, 2) == 2 * 10**6


def test_errors():
    with pytest.raises(ValueError):
        S.make_schedule(4, 5)
    with pytest.raises(ValueError):
        S.num_rounds(0, 1)
    with pytest.raises(ValueError):
        S.make_schedule(4, 0)


def test_native_equals_oracle_and_knows_closure_exhaustive():
    # acceptance 6: closure for every CN in [1, 64] and every fanout <= CN
    for cn in range(1, 65):
        for f in range(1, cn + 1):
            s = S.make_schedule(cn, f)
            assert s == osched.make_schedule(cn, f)
            assert len(s) == osched.num_rounds(cn, f)
            knows = osched.knows_closure(s, cn)
            assert all(len(k) == cn for k in knows), (cn, f)
            for rnd in s:
                for g, srcs in enumerate(rnd):
                    assert g not in srcs
            assert S.message_count_remote(s) <= S.message_count_paper(cn, f)


def test_power_of_radix_properties():
    # SPEC.md:187,241-242
    for r, cn in ((2, 16), (4, 16), (4, 64), (8, 64), (3, 27)):
        f = r
        s = S.make_schedule(cn, f)
        for rnd in s:
            assert all(len(srcs) == f - 1 for srcs in rnd)
        knows = [{g} for g in range(cn)]
        for i, rnd in enumerate(s):
            snap = [set(k) for k in knows]
            for g, srcs in enumerate(rnd):
                for x in srcs:
                    knows[g] |= snap[x]
            assert all(len(k) == r ** (i + 1) for k in knows)
        sends = [0] * cn
        for rnd in s:
            for srcs in rnd:
                for x in srcs:
                    sends[x] += 1
        recvs = [sum(len(rnd[g]) for rnd in s) for g in range(cn)]
        assert sends == recvs


def test_fanout_one_equals_two():
    for cn in range(2, 40):
        assert S.make_schedule(cn, 1) == S.make_schedule(cn, 2)
