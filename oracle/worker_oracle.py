"""TEST INFRASTRUCTURE ONLY (parity checker for csrc/k_worker.cu).

Python restatement of sched/worker.cpp: effective_priority (:11-14), form_batch (:16-37),
select_preemption_victim (:39-58).  Request ids are ranks in the ids' string order.
Python floats evaluate base + aging * (now - enqueue) in the reference's order, so every
comparison sees the same doubles; pinned against the compiled reference in
tests/test_worker.py."""
import functools


def effective_priority(base, enq, now, aging):
    return base + aging * (now - enq)


def form_batch(items, active_reservation, capacity, now, aging):
    """items: list of (base, enqueue, reservation, id_rank) -> admitted indices in order."""
    def cmp(a, b):
        ea = effective_priority(items[a][0], items[a][1], now, aging)
        eb = effective_priority(items[b][0], items[b][1], now, aging)
        if ea != eb:
            return -1 if ea > eb else 1
        if items[a][1] != items[b][1]:
            return -1 if items[a][1] < items[b][1] else 1
        return (items[a][3] > items[b][3]) - (items[a][3] < items[b][3])
    order = sorted(range(len(items)), key=functools.cmp_to_key(cmp))
    out, reserved = [], active_reservation
    for i in order:
        if reserved + items[i][2] > capacity:
            break
        reserved += items[i][2]
        out.append(i)
    return out


def preemption_victim(items, now, aging):
    v = 0
    ve = effective_priority(items[0][0], items[0][1], now, aging)
    for i in range(1, len(items)):
        e = effective_priority(items[i][0], items[i][1], now, aging)
        better = e < ve or (e == ve and items[i][1] > items[v][1]) or \
            (e == ve and items[i][1] == items[v][1] and items[i][3] > items[v][3])
        if better:
            v, ve = i, e
    return v
