"""Brute-force microsecond-stepping simulator — a pin for the oracle's DES.

Deliberately the dumbest possible algorithm: it walks simulated time one
microsecond at a time and, at every microsecond, applies the serving rules of
SPEC.md S:245 (continuous batching) in the order fixed by S:247 / readings
R6-R9: iteration end, prefill ends (by j), arrivals (by j), then — if the loop
is idle — ingest, admission and iteration start.  prof["prefill_mode"] = 1
(NEXT-4 contention): requests admitted at a boundary prefill inside the
next iteration, which lasts cost(B) + their prefill times (B = 0: just those).
prof["kv_policy"] = 1 (NEXT-4 preemption): admission needs only the current
context (input + words emitted) to fit kv_cap_words; at an iteration end whose
contexts exceed it, the latest admitted requests (while more than one is in the
system) go back to the front of the queue and later prefill input + emitted
again, that prefill's end emitting their next word.  No event heap, no
incremental sums (instants at which nothing is scheduled are skipped: every
rule fires only at an iteration end, a prefill end or an arrival).  Usable only on tiny traces (<= ~2e6 µs).  Controller:
every law recomputed here in exact rationals from its own per-second samples
(TBT gaps, or E2E / SLO of the completions, R3): MAP, STEP
(R5), MPC (R41), BBR (R42, delivery = decode words of the second), PCC (R43).
"""
from __future__ import annotations

from fractions import Fraction


class _Law:
    """The controller laws written out from their definitions,
    with Fraction arithmetic: one call per ingested second."""

    def __init__(self, law, t1, t2, r_min, r_max, window, rungs, horizon_s, w_lat, w_q, w_osc, step_bp):
        self.law, self.t1, self.t2, self.r_min, self.r_max, self.window = law, t1, t2, r_min, r_max, window
        self.rungs = list(rungs)
        if self.rungs:
            self.r_min, self.r_max = self.rungs[0], self.rungs[-1]
        self.h, self.w_lat, self.w_q, self.w_osc, self.step = horizon_s, w_lat, w_q, w_osc, step_bp
        self.samples, self.words = [], []
        self.r = 0
        self.active = False
        self.rung = 0
        self.rt_min = None
        self.phase, self.r_base, self.cost_a = 0, 0, None

    def ingest(self, x, w):
        self.samples.append(x)
        self.words.append(w)
        ys = self.samples[-self.window:]
        k = len(ys)
        ma = Fraction(sum(ys), k)
        prev_r, prev_active = self.r, self.active
        if self.law == "map":
            self.active = ma >= self.t1
            if self.active:
                r = min(self.r_max, int(Fraction(self.r_min) + Fraction(self.r_max - self.r_min) * (ma - self.t1)
                                        / (self.t2 - self.t1)))
                if self.rungs:
                    r = max([g for g in self.rungs if g <= r] or [self.rungs[0]])
                self.r = r
            else:
                self.r = 0
        elif self.law == "step":
            self.active = ma >= self.t1
            if self.active:
                self.rung = 0 if not prev_active else min(self.rung + 1, len(self.rungs) - 1)
                self.r = self.rungs[self.rung]
            else:
                self.r = 0
        elif self.law == "mpc":
            F = ma + (Fraction(self.h * (ys[-1] - ys[0]), k - 1) if k >= 2 else 0)
            F = max(F, Fraction(0))
            cands = [0] + (self.rungs if self.rungs else
                           [self.r_min + i * (self.r_max - self.r_min) // 30 for i in range(31)])
            best = None
            for c in cands:
                J = self.w_lat * max(Fraction(0), F * (1 - Fraction(c, 10000)) - self.t1) + self.w_q * c + \
                    self.w_osc * abs(c - prev_r)
                if best is None or J < best[0]:
                    best = (J, c)
            self.r = best[1]
            self.active = self.r > 0
        elif self.law == "bbr":
            self.rt_min = x if self.rt_min is None else min(self.rt_min, x)
            bw = max(self.words[-self.window:])
            congested = ma >= self.rt_min + self.t1
            plateau = Fraction(w) >= Fraction(7, 8) * bw
            if congested and plateau:
                if self.rungs:
                    self.rung = 0 if prev_r == 0 else min(self.rung + 1, len(self.rungs) - 1)
                    self.r = self.rungs[self.rung]
                else:
                    self.r = self.r_min if prev_r == 0 else min(self.r_max, prev_r + self.step)
            elif not congested:
                if self.rungs:
                    if prev_r == 0 or self.rung == 0:
                        self.r = 0
                    else:
                        self.rung -= 1
                        self.r = self.rungs[self.rung]
                else:
                    self.r = 0 if prev_r <= self.r_min else max(self.r_min, prev_r - self.step)
            self.active = self.r > 0
        elif self.law == "pcc":
            self.active = ma >= self.t1
            if not self.active:
                self.phase, self.r_base, self.r = 0, 0, 0
            else:
                cost = self.w_lat * max(0, x - self.t1) + self.w_q * prev_r
                if self.phase == 0:
                    self.r_base = self.r_min
                elif self.phase == 1:
                    self.cost_a = cost
                else:
                    if self.cost_a < cost:
                        self.r_base = min(self.r_max, self.r_base + self.step)
                    elif cost < self.cost_a:
                        self.r_base = max(self.r_min, self.r_base - self.step)
                if self.phase == 1:
                    self.r = max(self.r_min, self.r_base - self.step)
                    self.phase = 2
                else:
                    self.r = min(self.r_max, self.r_base + self.step)
                    self.phase = 1
        return self.r


def simulate(requests, prof, horizon_us, law="off", t1=0, t2=0, r_min=500, r_max=2000, window=5,
             r_const=0, mode_drain=True, rungs=(), horizon_s=0, w_lat=0, w_q=0, w_osc=0, step_bp=0,
             signal="tbt", slo_us=0):
    tpw = prof.get("tpw_q16", 0)

    def tok(w):  # NEXT-4 token-level costs (R44): round-half-up w * tpw, at least 1
        return w if not tpw else min(1 << 24, max(1, int(Fraction(w * tpw, 65536) + Fraction(1, 2))))

    requests = [dict(q, input=tok(q["input"])) for q in requests]  # the engine counts input tokens
    n = len(requests)
    st = ["future"] * n
    admit = [None] * n
    pend = [None] * n
    first = [None] * n
    done = [None] * n
    last = [None] * n
    emitted = [0] * n
    R = [0] * n
    rbp = [0] * n
    queue = []
    ready = []
    seq = [None] * n
    enq = [q["a_us"] for q in requests]
    next_seq = 0
    preemptions = 0
    recompute_words = 0
    sum_queue = 0
    preempt = prof.get("kv_policy", 0) == 1 and prof.get("kv_cap_words", 0) > 0
    in_system = ("prefill", "ready", "decoding", "pending")
    batch = []
    iter_end = None
    ticks = 0
    words_out = 0
    gaps = [[] for _ in range(n)]
    sec_sum, sec_cnt = {}, {}
    e2e_sum, e2e_cnt, slo_cnt = {}, {}, {}
    ctl = _Law(law, t1, t2, r_min, r_max, window, rungs, horizon_s, w_lat, w_q, w_osc, step_bp)

    def complete(m, t):
        st[m] = "done"
        done[m] = t
        e = t - requests[m]["a_us"]
        s_ = t // 10**6
        e2e_sum[s_] = e2e_sum.get(s_, 0) + e
        e2e_cnt[s_] = e2e_cnt.get(s_, 0) + 1
        slo_cnt[s_] = slo_cnt.get(s_, 0) + (1 if e > slo_us else 0)

    ingested_upto = 0  # next second to ingest
    r_cur = r_const if law == "const" else 0
    last_event = 0
    t = 0
    while t < horizon_us:
        anything = False
        if iter_end == t:
            anything = True
            for m in batch:
                g = t - last[m]
                gaps[m].append(g)
                sec_sum[t // 10**6] = sec_sum.get(t // 10**6, 0) + g
                sec_cnt[t // 10**6] = sec_cnt.get(t // 10**6, 0) + 1
                last[m] = t
                emitted[m] += 1
                words_out += 1
                if emitted[m] == R[m]:
                    complete(m, t)
                else:
                    st[m] = "ready"
                    ready.append(m)
            batch = []
            iter_end = None
            if preempt:  # contexts over the capacity: the latest admitted go back to the queue front
                while True:
                    inside = [i for i in range(n) if st[i] in in_system]
                    F = sum(requests[i]["input"] + emitted[i] for i in inside)
                    if F <= prof["kv_cap_words"] or len(inside) <= 1:
                        break
                    v = max(inside, key=lambda i: seq[i])
                    if v in ready:
                        ready.remove(v)
                    st[v] = "queued"
                    enq[v] = t
                    queue.insert(0, v)
                    preemptions += 1
        for m in range(n):
            if st[m] == "prefill" and pend[m] == t and emitted[m] > 0:  # recompute prefill: next word
                anything = True
                g = t - last[m]
                gaps[m].append(g)
                sec_sum[t // 10**6] = sec_sum.get(t // 10**6, 0) + g
                sec_cnt[t // 10**6] = sec_cnt.get(t // 10**6, 0) + 1
                last[m] = t
                emitted[m] += 1
                words_out += 1
                if emitted[m] == R[m]:
                    complete(m, t)
                else:
                    st[m] = "ready"
                    ready.append(m)
                continue
            if st[m] == "prefill" and pend[m] == t:
                anything = True
                first[m] = t
                last[m] = t
                emitted[m] = 1
                words_out += 1
                if R[m] == 1:
                    complete(m, t)
                else:
                    st[m] = "ready"
                    ready.append(m)
        for m in range(n):
            if st[m] == "future" and requests[m]["a_us"] == t:
                anything = True
                st[m] = "queued"
                queue.append(m)
        if anything:
            last_event = t
        if anything and iter_end is None:
            # ingest every closed second
            while (ingested_upto + 1) * 10**6 <= t:
                s = ingested_upto
                ingested_upto += 1
                if signal == "tbt":
                    num, den = sec_sum.get(s, 0), sec_cnt.get(s, 0)
                elif signal == "e2e":
                    num, den = e2e_sum.get(s, 0), e2e_cnt.get(s, 0)
                else:  # slo: per-mille of completions with E2E > slo_us
                    num, den = 1000 * slo_cnt.get(s, 0), e2e_cnt.get(s, 0)
                if den == 0:
                    continue
                if law in ("map", "step", "mpc", "bbr", "pcc"):
                    r_cur = ctl.ingest(num // den, sec_cnt.get(s, 0))
            in_sys = sum(1 for i in range(n) if st[i] in ("prefill", "ready", "decoding", "pending"))
            cap = prof.get("kv_cap_words", 0)
            while in_sys < prof["max_batch"] and queue:
                m = queue[0]
                q = requests[m]
                if preempt:
                    F = sum(requests[i]["input"] + emitted[i] for i in range(n) if st[i] in in_system)
                    ctx = q["input"] + emitted[m]
                    if in_sys > 0 and F + ctx > cap:
                        break
                    if admit[m] is not None:  # re-admission of a preempted request: R stays
                        queue.pop(0)
                        seq[m] = next_seq
                        next_seq += 1
                        sum_queue += t - enq[m]
                        recompute_words += ctx
                        pend[m] = t + max(1, prof["prefill_ns_per_word"] * ctx // 1000)
                        st[m] = "prefill"
                        in_sys += 1
                        continue
                elif cap:  # NEXT-4 KV-capacity admission: whole contexts must fit (empty system always admits)
                    if r_cur > 0:
                        Nh = max(1, int(Fraction(q.get("P", q["U"])) * (Fraction(10000 - r_cur, 10000)) + Fraction(1, 2)))
                        Rh = max(1, int(Fraction(Nh) * Fraction(q.get("fcomp_q16", 65536), 65536) + Fraction(1, 2)))
                    else:
                        Rh = q["U"]
                    Rh = tok(Rh)
                    reserved = sum(requests[i]["input"] + R[i] for i in range(n)
                                   if st[i] in ("prefill", "ready", "decoding", "pending"))
                    if in_sys > 0 and reserved + q["input"] + Rh > cap:
                        break
                queue.pop(0)
                admit[m] = t
                seq[m] = next_seq
                next_seq += 1
                sum_queue += t - enq[m]
                rbp[m] = r_cur
                q = requests[m]
                if r_cur > 0:
                    N = max(1, int(Fraction(q.get("P", q["U"])) * (Fraction(10000 - r_cur, 10000)) + Fraction(1, 2)))
                    R[m] = max(1, int(Fraction(N) * Fraction(q.get("fcomp_q16", 65536), 65536) + Fraction(1, 2)))
                else:
                    R[m] = q["U"]
                R[m] = tok(R[m])  # realized words decoded as tokens
                pf = max(1, prof["prefill_ns_per_word"] * q["input"] // 1000)
                if prof.get("prefill_mode", 0):
                    pend[m] = pf  # a duration until the iteration starts
                    st[m] = "pending"
                else:
                    pend[m] = t + pf
                    st[m] = "prefill"
                in_sys += 1
            waiting = [m for m in range(n) if st[m] == "pending"]
            if ready or waiting:
                B = len(ready)
                K = sum(requests[m]["input"] + emitted[m] for m in ready)
                d = 0 if B == 0 else prof["t0_us"] + prof["slope_us"] * max(0, B - prof["knee"]) + \
                    prof.get("kv_ns_per_word", 0) * K // 1000
                d += sum(pend[m] for m in waiting)
                for m in waiting:
                    pend[m] = t + d
                    st[m] = "prefill"
                batch = list(ready)
                for m in batch:
                    st[m] = "decoding"
                ready = []
                iter_end = t + d
                ticks += 1
        t += 1
        if mode_drain and all(s in ("done",) for s in st):
            break
        # no rule fires at an instant without a scheduled iteration end, prefill
        # end or arrival: jump over such instants (state is constant there)
        nxt = [iter_end] if iter_end is not None else []
        nxt += [pend[m] for m in range(n) if st[m] == "prefill"]
        nxt += [requests[m]["a_us"] for m in range(n) if st[m] == "future"]
        nxt = [x for x in nxt if x >= t]
        t = min(nxt) if nxt else horizon_us
    end = last_event if mode_drain and all(s == "done" for s in st) else horizon_us
    if mode_drain and all(s == "done" for s in st):
        # idle was counted through t = end inclusive of the final µs loop; recount up to end
        pass
    return dict(admit=admit, first=first, done=done, R=R, r_bp=rbp, gaps=gaps, ticks=ticks,
                words_out=words_out, end_us=end, served=sum(1 for s in st if s == "done"),
                preemptions=preemptions, recompute_words=recompute_words, sum_queue_us=sum_queue)


def simulate_replicas(requests, prof, horizon_us, law="off", t1=0, t2=0, r_min=500, r_max=2000, window=5,
                      r_const=0, rungs=(), horizon_s=0, w_lat=0, w_q=0, w_osc=0, step_bp=0):
    """NEXT-4 multi-replica routing (reading R45), brute force: prof["replicas"]
    engines of prof["max_batch"] slots share one FIFO queue.  At every instant
    where something happened and some replica has no iteration running, the
    closed seconds are ingested (TBT signal) and the arrived queue head goes to
    an idle replica with a free slot, chosen least-loaded (fewest requests in
    the replica, lowest index) or round robin (prof["route"] = 1); then every
    idle replica with decode-ready requests starts an iteration.  Drain mode."""
    tpw = prof.get("tpw_q16", 0)

    def tok(w):
        return w if not tpw else min(1 << 24, max(1, int(Fraction(w * tpw, 65536) + Fraction(1, 2))))

    requests = [dict(q, input=tok(q["input"])) for q in requests]
    n = len(requests)
    NR = max(1, prof.get("replicas", 1))
    st = ["future"] * n
    rep = [None] * n
    admit, pend, first, done, last = [None] * n, [None] * n, [None] * n, [None] * n, [None] * n
    emitted, R, rbp = [0] * n, [0] * n, [0] * n
    gaps = [[] for _ in range(n)]
    queue = []
    iter_end = [None] * NR
    batch = [[] for _ in range(NR)]
    rr = 0
    ticks = 0
    sec_sum, sec_cnt = {}, {}
    ctl = _Law(law, t1, t2, r_min, r_max, window, rungs, horizon_s, w_lat, w_q, w_osc, step_bp)
    r_cur = r_const if law == "const" else 0
    ingested_upto = 0
    last_event = 0
    t = 0
    while t < horizon_us:
        anything = False
        for q in range(NR):
            if iter_end[q] == t:
                anything = True
                for m in batch[q]:
                    g = t - last[m]
                    gaps[m].append(g)
                    sec_sum[t // 10**6] = sec_sum.get(t // 10**6, 0) + g
                    sec_cnt[t // 10**6] = sec_cnt.get(t // 10**6, 0) + 1
                    last[m] = t
                    emitted[m] += 1
                    if emitted[m] == R[m]:
                        st[m], done[m] = "done", t
                    else:
                        st[m] = "ready"
                batch[q] = []
                iter_end[q] = None
        for m in range(n):
            if st[m] == "prefill" and pend[m] == t:
                anything = True
                first[m] = last[m] = t
                emitted[m] = 1
                if R[m] == 1:
                    st[m], done[m] = "done", t
                else:
                    st[m] = "ready"
        for m in range(n):
            if st[m] == "future" and requests[m]["a_us"] == t:
                anything = True
                st[m] = "queued"
                queue.append(m)
        if anything:
            last_event = t
        idle = [q for q in range(NR) if iter_end[q] is None]
        if anything and idle:
            while (ingested_upto + 1) * 10**6 <= t:
                s = ingested_upto
                ingested_upto += 1
                if sec_cnt.get(s, 0) and law in ("map", "step", "mpc", "bbr", "pcc"):
                    r_cur = ctl.ingest(sec_sum[s] // sec_cnt[s], sec_cnt[s])
            while queue:
                load = {q: sum(1 for i in range(n) if rep[i] == q and st[i] in ("prefill", "ready", "decoding"))
                        for q in idle}
                ok = [q for q in idle if load[q] < prof["max_batch"]]
                if not ok:
                    break
                if prof.get("route", 0) == 1:
                    q = min(ok, key=lambda c: (c - rr) % NR)
                    rr = (q + 1) % NR
                else:
                    q = min(ok, key=lambda c: (load[c], c))
                m = queue.pop(0)
                rep[m] = q
                admit[m] = t
                rbp[m] = r_cur
                qq = requests[m]
                if r_cur > 0:
                    N = max(1, int(Fraction(qq.get("P", qq["U"])) * Fraction(10000 - r_cur, 10000) + Fraction(1, 2)))
                    R[m] = max(1, int(Fraction(N) * Fraction(qq.get("fcomp_q16", 65536), 65536) + Fraction(1, 2)))
                else:
                    R[m] = qq["U"]
                R[m] = tok(R[m])
                pend[m] = t + max(1, prof["prefill_ns_per_word"] * qq["input"] // 1000)
                st[m] = "prefill"
            for q in idle:
                mine = [m for m in range(n) if rep[m] == q and st[m] == "ready"]
                if mine:
                    B = len(mine)
                    K = sum(requests[m]["input"] + emitted[m] for m in mine)
                    d = prof["t0_us"] + prof["slope_us"] * max(0, B - prof["knee"]) + \
                        prof.get("kv_ns_per_word", 0) * K // 1000
                    for m in mine:
                        st[m] = "decoding"
                    batch[q] = mine
                    iter_end[q] = t + d
                    ticks += 1
        t += 1
        if all(s == "done" for s in st):
            break
        nxt = [e for e in iter_end if e is not None]
        nxt += [pend[m] for m in range(n) if st[m] == "prefill"]
        nxt += [requests[m]["a_us"] for m in range(n) if st[m] == "future"]
        nxt = [x for x in nxt if x >= t]
        t = min(nxt) if nxt else horizon_us
    return dict(admit=admit, first=first, done=done, R=R, r_bp=rbp, gaps=gaps, ticks=ticks, rep=rep,
                end_us=last_event if all(s == "done" for s in st) else horizon_us,
                served=sum(1 for s in st if s == "done"))
