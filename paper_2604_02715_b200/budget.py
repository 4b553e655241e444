"""Spending a fixed expert-HBM budget (BASELINE configs 2-5).

The reference holds a two-layer window and moves a device-resident fraction alpha of
the compressed experts (storage.py:143-168, simulate.py:50-66: window + alpha x
compressed pool must fit the device budget).  On a B200 three kinds of residency
compete for the same bytes:

* ring blocks (raw, `eb` bytes each): the window every streamed expert passes through;
  a sub-layer ring needs only 2 windows of w experts;
* device-tier experts (compressed, `ceb` ≈ 0.66 eb each): no PCIe traffic, but decoded on
  the GPU into the ring every step;
* pinned experts (raw, `eb` each): neither link nor decode cost.

`plan_residency` picks the ring, the device-tier and the pinned experts that minimise a
step-time model -- link time of the host-tier records vs decode plus compute on the SMs
-- under the budget.  It returns bool masks the runner applies (`StreamedRunner.apply_plan`).
Counts are balanced across layers; inside a layer the pinned experts sit at the end, and
the device-tier experts spread over the ring windows (each window mixes device- and
host-tier experts, so the link never idles on a window, while a window's host records
stay contiguous in the pool).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass
class ResidencyPlan:
    ring: int                 # ring blocks per kind (sub-layer ring when < depth x streamed experts)
    device_mask: np.ndarray   # bool [N][L]: compressed in HBM, decoded into the ring each step
    pinned_mask: np.ndarray   # bool [N][L]: raw, resident for good
    hbm_bytes: float          # ring + device tier + pinned (+ shared), the budget's numerator
    est_step_s: float         # modelled step time
    link_bytes: float         # host-tier record bytes per step
    depth: int = 2            # windows in flight on the ring (ring // depth experts each)
    decode_bytes: float = 0.0  # raw bytes the GPU decoder produces per step

    @property
    def device_experts(self) -> int:
        return int(self.device_mask.sum())

    @property
    def pinned_experts(self) -> int:
        return int(self.pinned_mask.sum())

    @property
    def fx4_experts(self) -> int:
        """Device-tier experts in FX4 records (mixed plans; all device-tier experts of FX4 plans)."""
        m = getattr(self, "fx4_mask", None)
        if m is not None:
            return int(m.sum())
        return self.device_experts if getattr(self, "device_format", None) == "fx4" else 0

    @property
    def host_experts(self) -> int:
        return int(self.device_mask.size - self.device_mask.sum() - self.pinned_mask.sum())


def _fill(total: int, caps) -> list:
    """`total` items over slots of capacity `caps`, as even as the capacities allow."""
    out = [0] * len(caps)
    left = min(int(total), int(sum(caps)))
    while left > 0:
        open_ = [j for j in range(len(caps)) if out[j] < caps[j]]
        share = max(1, left // len(open_))
        for j in open_:
            take = min(share, caps[j] - out[j], left)
            out[j] += take
            left -= take
            if left == 0:
                break
    return out


def _spread_row(streamed: int, m: int, window: int) -> np.ndarray:
    """m of the first `streamed` positions, spread over windows of `window`, contiguous inside."""
    row = np.zeros(streamed, dtype=bool)
    if m <= 0 or streamed <= 0:
        return row
    w = max(1, min(window, streamed))
    caps = [min(w, streamed - a) for a in range(0, streamed, w)]
    for j, n in enumerate(_fill(m, caps)):
        row[j * w:j * w + n] = True
    return row


def _spaced(total: int, N: int) -> list:
    """`total` items over N slots, the remainder spaced evenly (1 item over 8 slots: slot 4;
    3 over 8: slots 1, 4, 6), not bunched at one end."""
    base, rem = divmod(int(total), N)
    out = [base] * N
    for i in range(rem):
        out[int((i + 0.5) * N / rem)] += 1
    return out


def _balanced(total: int, N: int):
    return [(l + 1) * total // N - l * total // N for l in range(N)]


def plan_residency(N: int, L: int, eb: float, ceb: float, budget_bytes: float, *, shared_bytes: float = 0.0,
                   overhead_bytes: float = 0.0, b_link: float = 54e9, b_dec: float = 1100e9, t_compute: float = 0.0,
                   min_window_bytes: float = 128 * 2**20, allow_pinned: bool = True, depth: int | None = None,
                   window: int | None = None, dev_ceb: float | None = None, b_dev: float | None = None,
                   dev_fused: bool = False) -> ResidencyPlan:
    """Choose (ring, device tier, pinned) for N layers x L experts under `budget_bytes`.

    eb: raw bytes of one expert (both tensors); ceb: its compressed record bytes.
    overhead_bytes: HBM the codec holds for host-tier records (staging buffers, the device-resident
    chunk index): counted inside ``budget_bytes`` like the shared experts, so the plan's whole
    expert footprint stays within the budget -- unless the plan leaves no expert on the host
    tier, which releases them (``ResidencyPlan.host_experts == 0``).
    Step model: max(link_bytes / b_link, decoded_raw_bytes / b_dec + t_compute).
    dev_ceb / b_dev: HBM bytes and raw-equivalent rate of a device-tier expert when the device
    tier uses another record format than the host tier (FX4: larger records, faster decode);
    dev_fused: device-tier experts are read in place by the decode-into-GEMM kernel, so b_dev
    covers their GEMM too and they leave t_compute (which then is the resident step time).
    depth: windows in flight (the ring holds depth windows); window: experts per window
    (default: enough for min_window_bytes).  depth None: 1 when the plan is clearly
    link-bound (link time >= 1.5x decode time: the ring's second window buys nothing while
    the link is the bottleneck, and its bytes hold more device-tier experts -- Mixtral 50%:
    +10%), else 2 (decode-bound plans need the decode of window g+1 to overlap window g's
    compute -- DSv3 65%: depth 1 is 22% slower).
    """
    kw = dict(dev_ceb=dev_ceb, b_dev=b_dev, dev_fused=dev_fused)
    if depth is None:
        one = plan_residency(N, L, eb, ceb, budget_bytes, shared_bytes=shared_bytes, overhead_bytes=overhead_bytes,
                             b_link=b_link, b_dec=b_dec,
                             t_compute=t_compute, min_window_bytes=min_window_bytes, allow_pinned=allow_pinned,
                             depth=1, window=window, **kw)
        if one.ring and one.link_bytes / b_link >= 1.5 * one.decode_bytes / b_dec:
            return one
        return plan_residency(N, L, eb, ceb, budget_bytes, shared_bytes=shared_bytes, overhead_bytes=overhead_bytes,
                              b_link=b_link, b_dec=b_dec, t_compute=t_compute, min_window_bytes=min_window_bytes,
                              allow_pinned=allow_pinned, depth=2, window=window, **kw)
    dceb = ceb if dev_ceb is None else dev_ceb
    bdev = b_dec if b_dev is None else b_dev
    total = N * L
    cap = budget_bytes - shared_bytes - overhead_bytes
    if window is None:
        # one expert per window once it is >= min_window_bytes (Mixtral: ring 2 instead of 4
        # frees 0.7 GB for the device tier, +7% at 25%); smaller experts batch into windows
        # of >= min_window_bytes (DSv3's 88 MB experts: 2 per window, 1 measured 10-20% slower)
        window = int(max(1, -(-min_window_bytes // eb)))
    w_min = int(min(L, window))
    best = None
    # with the device tier read in place, pinned experts run in a second GEMM launch beside the
    # layer's decode-into-GEMM launch (two half-empty waves, no gate/up -> down overlap): measured
    # slower per expert than the FX4 experts they replace (Mixtral 90%, 27 pinned: 42.2 K tok/s vs
    # 45.3 K at 80% with 2, r2_t58), so fused plans pin whole layers only
    whole = dev_fused
    p_grid = (range(0, total + 1, L) if whole else range(0, total + 1)) if allow_pinned else [0]

    def layers_of(p):
        return [L * c for c in _spaced(p // L, N)] if whole else _balanced(p, N)

    for p in p_grid:
        p_layer = layers_of(p)
        streamed_max = L - min(p_layer)
        if streamed_max == 0:
            ring = 0
        elif dev_fused:
            # device-tier experts read in place hold no ring block: the ring serves the host
            # tier only (one window of it in flight when nothing else is on the host)
            d_max = int(min(total - p, max(0.0, cap - depth * eb - p * eb) // dceb))
            host_layer = -(-(total - p - d_max) // N)
            ring = depth * max(1, min(w_min, host_layer))
        else:
            ring = depth * min(w_min, streamed_max)
        room = cap - ring * eb - p * eb
        # with every streamed expert on the device tier nothing crosses the link, and the
        # codec's staging buffers and host chunk index (overhead_bytes) are released
        all_device = (total - p) * dceb <= room + overhead_bytes
        if all_device:
            room = max(room, (total - p) * dceb)
        if room < 0:
            continue
        # all_device: place every streamed expert (room // dceb can round (total - p) * dceb / dceb
        # down to total - p - 1, leaving one host expert whose overhead the room did not charge:
        # Qwen3 x 48 layers at 80% ran at a 0.819 footprint)
        d = total - p if all_device else int(min(total - p, room // dceb))
        link = (total - p - d) * ceb
        decode = (total - p) * eb
        sm = (total - p - d) * eb / b_dec + d * eb / bdev + t_compute * (1.0 - (d / total if dev_fused else 0.0))
        # a host record's transfer is only partly hidden when the SMs are the bottleneck: the
        # staging ring holds ~1 record ahead and a record is released when its window decodes
        # (measured: an SM-bound step exposes about half its link time, DESIGN §5 calibration)
        est = max(link / b_link, sm + HOST_EXPOSED * link / b_link)
        key = (est, -ring)
        if best is None or key < best[0]:
            best = (key, p, d, ring, link)
    if best is None:
        if w_min > 1:  # small experts: a narrower window still fits (tiny: 8 x 0.8 MB > 25%)
            return plan_residency(N, L, eb, ceb, budget_bytes, shared_bytes=shared_bytes,
                                  overhead_bytes=overhead_bytes, b_link=b_link, b_dec=b_dec, t_compute=t_compute, min_window_bytes=min_window_bytes,
                                  allow_pinned=allow_pinned, depth=depth, window=max(1, w_min // 2), **kw)
        raise ValueError(f"budget {budget_bytes:.3g} B cannot hold a ring")
    (est, _), p, d, ring, link = best
    p_layer = layers_of(p)
    # host-tier experts spaced evenly over the layers: each host record then has the
    # layers since the previous one to cross the link (the staging ring holds about one
    # record ahead), instead of queueing behind a neighbour (Mixtral 80%: 3 host experts
    # bunched in layers 1, 7, 8 stalled 1.8 ms per step)
    h_layer = _spaced(total - p - d, N)
    d_layer = [L - q - hh for q, hh in zip(p_layer, h_layer)]
    if min(d_layer) < 0:
        d_layer = _fill(d, [L - q for q in p_layer])
    pinned = np.zeros((N, L), dtype=bool)
    for l in range(N):
        if p_layer[l]:
            pinned[l, L - p_layer[l]:] = True
    device = np.zeros((N, L), dtype=bool)
    w = max(1, ring // depth) if ring else 1
    for l in range(N):
        streamed = L - p_layer[l]
        device[l, :streamed] = _spread_row(streamed, d_layer[l], w)
    hbm = ring * eb + p * eb + device.sum() * dceb + shared_bytes + (overhead_bytes if total - p - d else 0.0)
    return ResidencyPlan(ring, device, pinned, float(hbm), float(est), float(link), depth, float((total - p) * eb))


# Raw-equivalent rates the format choice is made with (B200 measurements, Mixtral T = 256,
# `calibrate`, profiles/r2_calibrate_mixtral_v2.json): the Huffman decoder expanding into the ring
# beside the GEMMs (raw bytes over the step time beyond resident compute), and
# the decode-into-GEMM kernel reading FX4 records through TMA-staged compressed stages (GEMM
# included: 4.28 TB/s raw-equivalent with the A tiles in TMEM, `calibrate` in r2_t58).  Resident GEMMs stream raw
# weights at about 5.2 TB/s.
B_DEC_HUFFMAN = 1.8e12
B_FUSED_FX4 = 4.2e12
B_RESIDENT = 5.2e12
HOST_EXPOSED = 0.5  # share of the host link time an SM-bound step cannot hide


def fx4_expert_bytes(H: int, F: int) -> float:
    """HBM bytes of one expert's FX4 records (fx4.cuh layout, no escapes)."""
    r16 = lambda x: (x + 15) // 16 * 16
    total = 0
    for n in (2 * H * F, F * H):
        total += r16(n) + r16(n // 2) + r16(4 * (n // 256 + 1)) + 16 + 256
    return float(total)


def plan_tiers(N: int, L: int, eb: float, ceb: float, budget_bytes: float, *, fx4_ceb: float | None = None,
               shared_bytes: float = 0.0, overhead_bytes: float = 0.0, b_link: float = 54e9,
               b_dec: float = B_DEC_HUFFMAN, b_fx4: float = B_FUSED_FX4, b_resident: float = B_RESIDENT,
               device_format: str = "auto", units_per_expert: int = 0, num_sms: int = 148,
               **kw) -> ResidencyPlan:
    """Plan the budget with the device tier in exponent-Huffman records (decoded into the ring)
    and, when fx4_ceb is given, in FX4 records read in place by the decode-into-GEMM kernel;
    return the plan whose modelled step is shorter, tagged with ``device_format`` and ``fused``.

    Both candidates are scored with one model: max(link time, SM time) where the SM time is
    the Huffman decode of every streamed expert that is not FX4-fused, the fused FX4 experts at
    b_fx4, and the resident GEMM time of the rest.  Huffman wins while the link dominates
    (its records are 13% smaller, so more experts stay off the link); FX4 wins once the step
    is SM-bound."""
    t_res = N * L * eb / b_resident
    cands = []
    if device_format in ("auto", "huffman"):
        p = plan_residency(N, L, eb, ceb, budget_bytes, shared_bytes=shared_bytes, overhead_bytes=overhead_bytes,
                           b_link=b_link, b_dec=b_dec, t_compute=t_res, **kw)
        p.device_format, p.fused = "huffman", False
        cands.append(p)
    if fx4_ceb and device_format in ("auto", "fx4"):
        # the fused GEMM of a window has (experts per window) x units_per_expert units of work
        # (gate/up: F / 128 weight-row tiles); a window of fewer units than SMs leaves SMs idle
        # (DSv3's 2-expert windows: 32 units -> 8.6 K tok/s at 80% instead of the planned 33 K),
        # so FX4 plans also try windows wide enough to fill the GPU, at the rate the width allows
        widths = [kw.get("window")]
        if units_per_expert and not kw.get("window"):
            widths.append(max(1, min(L, -(-num_sms // units_per_expert))))
        for w in widths:
            fill = min(1.0, (w or 1) * units_per_expert / num_sms) if units_per_expert else 1.0
            kww = dict(kw, window=w)
            try:
                p = plan_residency(N, L, eb, ceb, budget_bytes, shared_bytes=shared_bytes,
                                   overhead_bytes=overhead_bytes, b_link=b_link, b_dec=b_dec, t_compute=t_res,
                                   dev_ceb=fx4_ceb, b_dev=b_fx4 * fill, dev_fused=True, **kww)
            except ValueError:
                continue
            p.device_format, p.fused, p.fx4_rate = "fx4", True, b_fx4 * fill
            cands.append(p)

    if fx4_ceb and device_format in ("auto", "mixed"):
        p = _plan_mixed(N, L, eb, ceb, fx4_ceb, budget_bytes, shared_bytes=shared_bytes, b_dec=b_dec, b_fx4=b_fx4,
                        t_res=t_res, window=kw.get("window"), allow_pinned=kw.get("allow_pinned", True))
        if p is not None:
            cands.append(p)

    def score(p):
        total = N * L
        d, pin = p.device_experts, p.pinned_experts
        host = total - d - pin
        link = p.link_bytes / b_link
        if p.fused == 2:
            x = p.fx4_experts
            sm = (d - x) * eb / b_dec + x * eb / p.fx4_rate + t_res * (total - x) / total
        elif p.fused:
            sm = host * eb / b_dec + d * eb / p.fx4_rate + t_res * (total - d) / total
        else:
            sm = (host + d) * eb / b_dec + t_res
        return max(link, sm + HOST_EXPOSED * link)

    best = min(cands, key=score)
    best.est_step_s = score(best)
    return best


def _plan_mixed(N: int, L: int, eb: float, ceb: float, fx4_ceb: float, budget_bytes: float, *, shared_bytes: float,
                b_dec: float, b_fx4: float, t_res: float, window: int | None = None, allow_pinned: bool = True,
                min_window_bytes: float = 128 * 2**20):
    """A mixed device tier: every streamed expert on the device tier, as many as fit in FX4
    records (read in place by the decode-into-GEMM kernel, no ring block) and the rest in the
    denser exponent-Huffman records (decoded into a two-window ring).  Nothing crosses the link,
    so the host staging is released.  Fills the budgets between "all Huffman on the device tier"
    and "all FX4 on the device tier", where the single-format plans leave experts on the host
    tier (Mixtral 75%: 3 host experts in FX4 plans, all 256 on the device tier here).  None when
    the budget cannot hold every streamed expert in Huffman records."""
    total = N * L
    cap = budget_bytes - shared_bytes
    w = int(window or max(1, -(-min_window_bytes // eb)))
    step = fx4_ceb - ceb
    if step <= 0:
        return None
    best = None
    # pinned experts in whole layers only, as in the fused plans (plan_residency)
    whole_layers = lambda p: [L * c for c in _spaced(p // L, N)]
    for p in (range(0, total + 1, L) if allow_pinned else [0]):
        p_layer = whole_layers(p)
        S = total - p
        if S == 0:
            break
        # x FX4 experts; the ring holds two windows of the busiest layer's Huffman experts
        room0 = cap - p * eb - S * ceb
        x = int(min(S, (room0 - 2 * min(w, L) * eb) // step))
        if x < 0:
            continue
        h_layer = _spaced(S - x, N)
        ring = 2 * min(w, max(h_layer))
        if ring < 2 * min(w, L):  # few Huffman experts per layer: a smaller ring, more FX4
            x = int(min(S, (room0 - ring * eb) // step))
            h_layer = _spaced(S - x, N)
            ring = 2 * min(w, max(h_layer))
        if S - x <= 0:
            continue  # all FX4: the FX4 plan covers it
        sm = (S - x) * eb / b_dec + x * eb / b_fx4 + t_res * (total - x) / total
        key = (sm, -x)
        if best is None or key < best[0]:
            best = (key, p, x, ring, h_layer)
    if best is None:
        return None
    (est, _), p, x, ring, h_layer = best
    p_layer = whole_layers(p)
    pinned = np.zeros((N, L), dtype=bool)
    device = np.zeros((N, L), dtype=bool)
    fx4 = np.zeros((N, L), dtype=bool)
    for l in range(N):
        streamed = L - p_layer[l]
        if p_layer[l]:
            pinned[l, streamed:] = True
        device[l, :streamed] = True
        # Huffman experts first, FX4 after: the layer's last window is one wide decode-into-GEMM
        # launch over every FX4 expert, beside which the next layer's first Huffman decodes run
        # (Mixtral 75%: 17.4 K tok/s; Huffman experts spread one per window, each window then
        # a 1-expert fused launch: 14.5 K -- profiles/r2_mixed_layout_ab.jsonl)
        h = min(h_layer[l], streamed)
        fx4[l, :streamed] = True
        if os.environ.get("XPGB_MIXED_LAYOUT") == "spread":  # A/B only
            for i in range(h):
                fx4[l, int((i + 0.5) * streamed / h)] = False
        else:
            fx4[l, :h] = False
    x = int(fx4.sum())
    hbm = ring * eb + p * eb + x * fx4_ceb + (device.sum() - x) * ceb + shared_bytes
    plan = ResidencyPlan(ring, device, pinned, float(hbm), float(est), 0.0, 2, float((total - p) * eb))
    plan.device_format, plan.fused, plan.fx4_rate, plan.fx4_mask = "mixed", 2, b_fx4, fx4
    return plan
