"""NCCL matching rules over per-rank schedules recorded by dry-run decomposed handles
(stokes_dist_schedule; used by tests/test_gpu_nccl_schedule.py, pinned on synthetic schedules
by tests/test_nccl_schedule_checker.py).  No torch, no GPU."""
from collections import defaultdict

from paper_2603_14040_b200.decomp import tile_of

GSTART, GEND, SEND, RECV, ALLGATHER, ALLREDUCE, BODY, BODY_END = 1, 2, 3, 4, 5, 6, 7, 8


def steps_of(log):
    """[(kind, payload)]: ("p2p", [(op, peer, count, dtype)]) per group, ("coll", signature)."""
    out, cur = [], None
    for op, peer, cnt, dt, red in log:
        if op in (BODY, BODY_END):
            assert cur is None, "capture marker inside a group"
            out.append(("mark", (op, peer)))
        elif op == GSTART:
            assert cur is None, "nested group"
            cur = []
        elif op == GEND:
            assert cur is not None, "group end without start"
            out.append(("p2p", cur))
            cur = None
        elif op in (SEND, RECV):
            assert cur is not None, "point-to-point call outside a group"
            cur.append((op, peer, cnt, dt))
        else:
            assert op in (ALLGATHER, ALLREDUCE), op
            assert cur is None, "collective inside a group"
            out.append(("coll", (op, cnt, dt, red)))
    assert cur is None, "unterminated group"
    return out


def check_schedules(logs, px, py):
    """NCCL's matching rules over the ranks' recorded schedules; returns a summary."""
    n = px * py
    steps = [steps_of(lg) for lg in logs]
    assert len({len(s) for s in steps}) == 1, [len(s) for s in steps]
    nsend = ncoll = 0
    for k in range(len(steps[0])):
        kinds = {steps[r][k][0] for r in range(n)}
        assert len(kinds) == 1, (k, kinds)
        if steps[0][k][0] in ("coll", "mark"):
            sigs = {steps[r][k][1] for r in range(n)}
            assert len(sigs) == 1, (k, sigs)
            ncoll += steps[0][k][0] == "coll"
            continue
        sends, recvs = defaultdict(list), defaultdict(list)
        for r in range(n):
            tx, ty = tile_of(r, px, py)
            for op, peer, cnt, dt in steps[r][k][1]:
                qx, qy = tile_of(peer, px, py)
                assert peer != r and max(abs(qx - tx), abs(qy - ty)) == 1, (k, r, peer)  # sides + diagonals
                if op == SEND:
                    sends[(r, peer)].append((cnt, dt))
                    nsend += 1
                else:
                    recvs[(peer, r)].append((cnt, dt))  # keyed (sender, receiver)
        assert dict(sends) == dict(recvs), (k, dict(sends), dict(recvs))
    # one plain Uzawa iteration = the body captured between the markers (parity 0)
    per_it = None
    kinds = [s[0] for s in steps[0]]
    if ("mark", (BODY, 0)) in steps[0]:
        a = steps[0].index(("mark", (BODY, 0)))
        b = steps[0].index(("mark", (BODY_END, 0)))
        body = steps[0][a + 1:b]
        per_it = {"p2p_rounds": sum(1 for s in body if s[0] == "p2p"),
                  "p2p_rounds_with_traffic_rank0": sum(1 for s in body if s[0] == "p2p" and s[1]),
                  "collectives": [s[1] for s in body if s[0] == "coll"]}
    return {"steps": len(kinds), "p2p_rounds": kinds.count("p2p"), "collectives": ncoll,
            "sends_all_ranks": nsend, "calls_rank0": len(logs[0]), "per_iteration": per_it}
