"""Static nF1B event order and a dependency-driven executor (TEST INFRASTRUCTURE ONLY).

Paper passages:
  * nF1B: each mini-batch is split into m micro-batches; a stage runs the m
    micro-batch forwards and ONE collective backward for the mini-batch;
    scheduling avoids circular waiting between the passes.
  * the first node gets the data, each node forwards its output to the next,
    the loss is computed at the last node and the backward runs in reverse.
  * weights are updated after every mini-batch.

Readings:
  * Z6: stage s (0-based) keeps K_s = min(S - s, M) mini-batches in flight.
  * Z7: the order is STATIC: F(0..K-1, all micro), then for j = 0..M-1:
        B(j), U(j), then F(j+K, all micro) if j+K < M.
    It is timing-independent, so the versions each pass uses are reproducible.

`stage_order` writes that rule down.  `execute` is a different mechanism: a
round-robin over stages that fires a stage's next event only when its
cross-stage dependency has fired, asserts no deadlock, and counts the
stage-local weight versions (the update counter) each pass sees.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Event:
    kind: str          # "F" (micro-batch forward), "B" (mini-batch backward), "U" (update)
    mb: int            # mini-batch index j (0-based)
    micro: int = -1    # micro-batch index a for "F"; -1 otherwise


def inflight(S: int, s: int, M: int, K: int = 0) -> int:
    """K_s = min(S - s, M) (reading Z6).  K > 0 overrides S - s for a ONE-stage pipeline
    (tps_config.max_inflight): a single stage keeping K mini-batches in flight, i.e. the
    staleness a stage at depth K sees (the staleness sweep of BASELINE.json configs[1])."""
    if K:
        assert S == 1, "an in-flight override is defined for S = 1 only"
        return min(K, M)
    return min(S - s, M)


def stage_order(S: int, s: int, m: int, M: int, K: int = 0) -> list[Event]:
    """Static per-stage event list L_s (reading Z7; SURVEY Appendix A rule)."""
    K = inflight(S, s, M, K)
    ev: list[Event] = []
    for j in range(K):
        ev += [Event("F", j, a) for a in range(m)]
    for j in range(M):
        ev.append(Event("B", j))
        ev.append(Event("U", j))
        if j + K < M:
            ev += [Event("F", j + K, a) for a in range(m)]
    return ev


@dataclass
class TraceRow:
    stage: int
    kind: str
    mb: int
    micro: int
    v_used: int        # version the pass read (F: latest at forward; B: version its forward used)
    v_latest: int      # stage's latest version when the pass ran
    delta: int         # B only: v_latest - v_used (reading Z5); 0 otherwise


def execute(S: int, m: int, M: int, K: int = 0) -> tuple[list[tuple[int, Event]], list[TraceRow]]:
    """Dependency-driven replay of all stages' static orders.

    Dependencies: F(j,a)@s needs F(j,a)@s-1; B(j)@s needs B(j)@s+1
    (the last stage needs its own F(j, m-1), implied by its order); U(j) follows
    B(j) on the same stage.  Returns the global firing order and the trace.
    """
    orders = [stage_order(S, s, m, M, K) for s in range(S)]
    ptr = [0] * S
    done: set[tuple[int, Event]] = set()
    version = [0] * S                       # stage-local update counter
    fwd_version: dict[tuple[int, int], int] = {}
    fired: list[tuple[int, Event]] = []
    trace: list[TraceRow] = []
    total = sum(len(o) for o in orders)
    while len(fired) < total:
        progress = False
        for s in range(S):
            if ptr[s] >= len(orders[s]):
                continue
            e = orders[s][ptr[s]]
            if e.kind == "F" and s > 0 and (s - 1, e) not in done:
                continue
            if e.kind == "B" and s < S - 1 and (s + 1, e) not in done:
                continue
            # fire
            if e.kind == "F":
                prev = fwd_version.setdefault((s, e.mb), version[s])
                assert prev == version[s], "micro-batches of one mini-batch saw different versions"
                trace.append(TraceRow(s, "F", e.mb, e.micro, version[s], version[s], 0))
            elif e.kind == "B":
                vf = fwd_version[(s, e.mb)]
                trace.append(TraceRow(s, "B", e.mb, -1, vf, version[s], version[s] - vf))
            else:
                trace.append(TraceRow(s, "U", e.mb, -1, version[s], version[s], 0))
                version[s] += 1
            done.add((s, e))
            fired.append((s, e))
            ptr[s] += 1
            progress = True
        if not progress:
            raise RuntimeError("deadlock: no stage can fire its next event")
    return fired, trace
