"""Per-chunk timeline of SemOperator.apply_host on config 2: timing events around each
chunk's H2D, kernels and D2H on their streams, relative to one start event (ms).
Diagnostic only: re-issues the streamer's own schedule with extra events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_01422_b200 import configs  # noqa: E402
from paper_1806_01422_b200.ops import HostStreamer  # noqa: E402


def run(st, uh, vh, wh, outs, align=False, kernels=True, deps=True):
    ins = {"u": uh, "v": vh, "w": wh}
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t0 = E()
    cur = torch.cuda.current_stream()
    t0.record(cur)
    st.s_h2d.wait_stream(cur)
    S = st.nslots
    marks = []
    ev_in, ev_out, ev_free = [], [], []
    for c, p in enumerate(st.parts):
        slot = c % S
        op = st.ops[c]
        pad = (-p.gl * p.N) % 16 if align else 0   # owned slice 128-byte aligned
        m = {k: E() for k in ("h0", "h1", "c0", "c1", "d0", "d1")}
        with torch.cuda.stream(st.s_h2d):
            if c >= S and deps:
                st.s_h2d.wait_event(ev_free[c - S])
            m["h0"].record(st.s_h2d)
            for name in ("u", "v", "w"):
                dst = st._buf(slot, name)[pad:]
                for off, g, ln in st._ranges(p):
                    dst[off:off + ln].copy_(ins[name][g:g + ln], non_blocking=True)
            m["h1"].record(st.s_h2d)
            ev_in.append(m["h1"])
        with torch.cuda.stream(st.s_cmp):
            if deps:
                st.s_cmp.wait_event(ev_in[c])
            m["c0"].record(st.s_cmp)
            n = p.ext_ndof
            b = lambda k: st._buf(slot, k)[pad:pad + n]  # noqa: E731
            ub = b("u")
            if kernels:
                op.launch_rhs(ub, b("o_rhs"))
                op.launch_jac(ub, b("v"), b("o_jac"))
                op.launch_jact(ub, b("w"), b("o_jact"))
            m["c1"].record(st.s_cmp)
            ev_out.append(m["c1"])
        with torch.cuda.stream(st.s_d2h):
            if deps:
                st.s_d2h.wait_event(ev_out[c])
            m["d0"].record(st.s_d2h)
            sl = p.owned_slice()
            for k in ("rhs", "jac", "jact"):
                outs[k][p.g_lo:p.g_lo + p.n_own].copy_(st._buf(slot, "o_" + k)[pad:][sl], non_blocking=True)
            m["d1"].record(st.s_d2h)
            ev_free.append(m["d1"])
        marks.append(m)
    cur.wait_stream(st.s_d2h)
    torch.cuda.synchronize()
    return [{k: round(t0.elapsed_time(v), 3) for k, v in m.items()} for m in marks]


def main():
    c = configs.CFG2
    op = configs.cfg_operator(c, device="cuda:0")
    u, v, w = configs.operator_inputs(op.ndof, c["seed"])
    uh, vh, wh = (torch.from_numpy(a).pin_memory() for a in (u, v, w))
    outs = {k: torch.empty(op.ndof, dtype=torch.float64).pin_memory() for k in ("rhs", "jac", "jact")}
    for kern, deps in ((True, True), (False, True), (True, False), (False, False), (True, True)):
        st = HostStreamer(op, 8, 3)
        run(st, uh, vh, wh, outs, False, kern, deps)
        tl = run(st, uh, vh, wh, outs, False, kern, deps)
        print(json.dumps({"kernels": kern, "deps": deps, "timeline_ms": tl}), flush=True)


if __name__ == "__main__":
    main()
