"""program emission (emitter.py) and the execution model
(simulator.py) against the reference's own emitter / simulator (oracle/_ref,
the unmodified reference package built in this container): identical
programs, FIFO consistency, inference lowering, JSON round trip, and
identical simulation reports (makespan, busy / idle / comm-wait, peak
memory, deadlock diagnosis and the full event trace)."""

import pytest

from test_extension_validate import NAMES, _searched

ref = pytest.importorskip("oracle").load_reference()
pytestmark = pytest.mark.skipif(ref is None, reason="reference not built (oracle/build_ref.sh)")


def _ref_schedule(p, s):
    from repsched import placement as RP
    from repsched import schedule as RS

    from paper_2311_15269_b200.placement import placement_to_dict

    rp = RP.placement_from_dict(placement_to_dict(p))
    info = None if s.repetend is None else RS.RepetendInfo(
        s.repetend.start, s.repetend.end, s.repetend.period, s.repetend.nr)
    return RS.Schedule(rp, s.num_microbatches,
                       {RP.BlockInstance(b.stage, b.mb): t for b, t in s.entries.items()}, info)


def _as_dicts(progs):
    return [[x.to_dict() for x in prog] for prog in progs.programs]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("mode", ["nonblocking", "blocking"])
def test_emit_and_simulate_match_reference(name, mode):
    from repsched import emitter as RE
    from repsched import simulator as RSim

    from paper_2311_15269_b200 import emitter as E
    from paper_2311_15269_b200 import simulator as S
    from paper_2311_15269_b200.extension import extend

    p, s0 = _searched(name)
    for n in (s0.num_microbatches, s0.num_microbatches + 3):
        s = extend(s0, n)
        mine, theirs = E.emit(s, mode), RE.emit(_ref_schedule(p, s), mode)
        assert _as_dicts(mine) == _as_dicts(theirs)
        assert E.fifo_consistent(mine) == RE.fifo_consistent(theirs) is True
        assert _as_dicts(E.drop_backward(mine)) == _as_dicts(RE.drop_backward(theirs))
        back = E.programs_from_dict(E.programs_to_dict(mine))
        assert _as_dicts(back) == _as_dicts(mine)
        for cost in (0, 2):
            a = S.simulate(mine, S.SimConfig(comm_cost=cost, trace=True))
            b = RSim.simulate(theirs, RSim.SimConfig(comm_cost=cost, trace=True))
            assert (a.makespan, a.busy, a.idle, a.wait_comm, a.peak_memory, a.deadlock,
                    a.blocked, a.trace) == (b.makespan, b.busy, b.idle, b.wait_comm,
                                            b.peak_memory, b.deadlock, b.blocked, b.trace)


def test_deadlock_and_malformed_programs_match_reference():
    from repsched import emitter as RE
    from repsched import simulator as RSim

    from paper_2311_15269_b200 import emitter as E
    from paper_2311_15269_b200 import simulator as S

    p, s = _searched("x4_demo_k3")
    for mode in ("blocking", "nonblocking"):
        mine, theirs = E.emit(s, mode), RE.emit(_ref_schedule(p, s), mode)
        # swap the first two sends of a device with two: breaks the FIFO order
        dev = next(d for d, prog in enumerate(mine.programs)
                   if sum(x.op == "send" for x in prog) >= 2)
        for progs in (mine.programs, theirs.programs):
            idx = [k for k, x in enumerate(progs[dev]) if x.op == "send"][:2]
            progs[dev][idx[0]], progs[dev][idx[1]] = progs[dev][idx[1]], progs[dev][idx[0]]
        assert E.fifo_consistent(mine) == RE.fifo_consistent(theirs)
        a, b = S.simulate(mine), RSim.simulate(theirs)
        assert (a.deadlock, a.blocked, a.makespan) == (b.deadlock, b.blocked, b.makespan)
    mine = E.emit(s, "blocking")
    prog = next(pr for pr in mine.programs if any(x.op == "recv" for x in pr))
    prog.remove(next(x for x in prog if x.op == "recv"))
    with pytest.raises(S.MalformedProgram):
        S.simulate(mine)
