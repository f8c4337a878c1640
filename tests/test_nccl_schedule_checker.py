"""Pins of the NCCL schedule checker (tests/nccl_schedule_check.py) on synthetic schedules, on
the CPU: it must accept a valid multi-rank schedule and reject each way one can go wrong --
so that a green tests/test_gpu_nccl_schedule.py means the dry-run schedules really pair up.
A record is (op, peer, count, datatype, reduction) as stokes_dist_schedule writes it."""
import pytest

from nccl_schedule_check import ALLGATHER, ALLREDUCE, BODY, BODY_END, GEND, GSTART, RECV, SEND, check_schedules

D = 7  # ncclFloat64 (any value: only equality matters)


def grp(*ops):
    return [(GSTART, -1, 0, -1, -1), *ops, (GEND, -1, 0, -1, -1)]


def snd(peer, n):
    return (SEND, peer, n, D, -1)


def rcv(peer, n):
    return (RECV, peer, n, D, -1)


AR = (ALLREDUCE, -1, 3, D, 0)
AG = (ALLGATHER, -1, 100, D, -1)


def valid_2x1():
    r0 = grp(snd(1, 10), rcv(1, 10)) + [AR] + [(BODY, 0, 0, -1, -1)] + grp(snd(1, 4), snd(1, 6), rcv(1, 5)) + [AG] + [
        (BODY_END, 0, 0, -1, -1)]
    r1 = grp(rcv(0, 10), snd(0, 10)) + [AR] + [(BODY, 0, 0, -1, -1)] + grp(rcv(0, 4), snd(0, 5), rcv(0, 6)) + [AG] + [
        (BODY_END, 0, 0, -1, -1)]
    return [r0, r1]


def test_accepts_a_valid_schedule():
    s = check_schedules(valid_2x1(), 2, 1)
    assert s["p2p_rounds"] == 2 and s["collectives"] == 2 and s["sends_all_ranks"] == 5
    assert s["per_iteration"]["p2p_rounds"] == 1 and len(s["per_iteration"]["collectives"]) == 1


def test_accepts_diagonal_neighbours():
    # 2 x 2: rank 0 <-> rank 3 are diagonal neighbours (one-round exchange)
    logs = [grp(snd(3, 4), rcv(3, 4)), grp(), grp(), grp(snd(0, 4), rcv(0, 4))]
    check_schedules(logs, 2, 2)


@pytest.mark.parametrize("mutate", ["count", "missing_recv", "order", "collective", "steps", "outside_group",
                                    "self", "far_peer", "group_kind"])
def test_rejects(mutate):
    logs = valid_2x1()
    px = 2
    if mutate == "count":  # a receive of another size
        logs[1][1] = rcv(0, 11)
    elif mutate == "missing_recv":
        del logs[1][1]
    elif mutate == "order":  # two sends to the same peer received in the other order
        i = logs[1].index(rcv(0, 4))
        j = logs[1].index(rcv(0, 6))
        logs[1][i], logs[1][j] = logs[1][j], logs[1][i]
    elif mutate == "collective":  # all-reduce of another length on one rank
        logs[1][logs[1].index(AR)] = (ALLREDUCE, -1, 4, D, 0)
    elif mutate == "steps":  # one rank issues an extra collective
        logs[0].append(AR)
    elif mutate == "outside_group":
        logs[0].insert(0, snd(1, 1))
        logs[1].insert(0, rcv(0, 1))
    elif mutate == "self":
        logs[0][1] = snd(0, 10)
    elif mutate == "far_peer":  # 3 x 1: ranks 0 and 2 are not neighbours
        logs = [grp(snd(2, 1), rcv(2, 1)), grp(), grp(snd(0, 1), rcv(0, 1))]
        px = 3
    elif mutate == "group_kind":  # a p2p round on one rank where the other has a collective
        logs[1][logs[1].index(AR)] = (GSTART, -1, 0, -1, -1)
        logs[1].insert(logs[1].index((GSTART, -1, 0, -1, -1), 4) + 1, (GEND, -1, 0, -1, -1))
    with pytest.raises(AssertionError):
        check_schedules(logs, px, 1)
