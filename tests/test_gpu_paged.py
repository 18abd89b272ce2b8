"""The paged device KV store and the KvLedger byte accounting (SURVEY §8 a15,
f2; memsim.hpp:77-215) against the reference's own KvLedger (oracle/_ref,
driven with the engine's action order: engine.hpp:686-716, then store_new).

* byte totals after every step equal the reference ledger's;
* the device capacity check raises OutOfDeviceMemory at the same step with
  the reference's message (memsim.hpp:193-200);
* a paged cache whose pool is below the full KV decodes a three-phase
  schedule bit-identically to the dense-layout cache (offload / erase free
  slots, reload / restore / store_new take them), with poisoned offloads
  proving every gathered row was resident (engine.hpp:625-628);
* INT8 caches recompute deleted tokens with the fake-quant re-applied
  (engine.hpp:729-730).
"""
import numpy as np
import pytest
import torch

from oracle import Oracle, OutOfDeviceMemory, RefLedger, reference_available

pytestmark = pytest.mark.gpu
NAMES = ("offload", "delete", "reload", "recompute")


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available()
    from paper_2403_17312_b200 import api as a

    a.lib()
    return a


@pytest.fixture(scope="module")
def ref():
    if not reference_available():
        pytest.skip("oracle/_ref (the compiled reference) is absent")
    return Oracle("reference")


def ref_step(ref_oracle, led, plan, j, sels, k, L, s, steps, n_new, e):
    """Engine::decode_step's ledger work for step j on every layer, in order:
    step_actions against the ledger, apply_actions, store_new (engine.hpp:592-616)."""
    for l in range(L):
        tiers = led.tiers(l, n_new)
        acts = ref_oracle.step_actions(plan, j, sels[l], k, tiers, L, l, s, steps)
        if len(acts["offload"]):
            led.op("offload", l, acts["offload"])
        if len(acts["delete"]):
            led.op("erase", l, acts["delete"])
        if len(acts["reload"]):
            led.op("reload", l, acts["reload"])
        if len(acts["recompute"]):
            led.op("restore", l, acts["recompute"], e)
        led.op("store_new", l, [n_new], e)


def make_inputs(B, H, D, s, steps, seed, L):
    g = torch.Generator(device="cuda").manual_seed(seed)
    h = H * D
    ncap = s + steps + 2
    x = [torch.randn((B, ncap, h), generator=g, device="cuda").half() for _ in range(L)]
    wk = [(torch.randn((h, h), generator=g, device="cuda") / h ** 0.5).half() for _ in range(L)]
    wv = [(torch.randn((h, h), generator=g, device="cuda") / h ** 0.5).half() for _ in range(L)]
    kv = [((x[l].float() @ wk[l].float()).half().reshape(B, ncap, H, D),
           (x[l].float() @ wv[l].float()).half().reshape(B, ncap, H, D)) for l in range(L)]
    qs = [torch.randn((L, B, H, D), generator=g, device="cuda").half() * 2 for _ in range(steps + 1)]
    return x, wk, wv, kv, qs, ncap


def run_decode(api, cache, kv, qs, s, steps, r, L, check=None):
    B = kv[0][0].shape[0]
    H, D = kv[0][0].shape[2], kv[0][0].shape[3]
    outs = []
    out = torch.empty((L, B, H, D), device="cuda", dtype=torch.float16)
    for j in range(steps):
        n = s + j + 1
        kn = torch.stack([kv[l][0][:, n - 1] for l in range(L)]).contiguous()
        vn = torch.stack([kv[l][1][:, n - 1] for l in range(L)]).contiguous()
        cache.swa_decode_step(n, r, qs[j + 1], kn, vn, out)
        outs.append(out.clone())
        if check:
            check(j, n)
    return outs


def setup_cache(api, cache, kv, x, wk, wv, qs, s, L, recompute=True):
    for l in range(L):
        cache.append_tokens(l, 0, 0, kv[l][0][:, :s].contiguous(), kv[l][1][:, :s].contiguous())
        cache.prefill_seed(l, s, qs[0][l].contiguous())
        if recompute:
            cache.attach_recompute(l, x[l], wk[l], wv[l])


@pytest.mark.parametrize("extra", [0, 1])
def test_paged_ledger_totals_and_oom_match_reference(api, ref, extra):
    """Phase I only (no offloading): the device capacity runs out while the
    decode grows the KV. Totals agree with the reference KvLedger after every
    step, and OutOfDeviceMemory surfaces at the reference's step (the device
    ledger runs one step ahead, so the failure of step j shows after call
    j - 1). With a budget that is a multiple of L x B token entries the
    message is the reference's own; with one entry more (extra = 1) the pool,
    split evenly over (layer, sequence), fills on one layer before the global
    count does: the same step fails as a pool exhaustion."""
    L, B, H, D, s, steps, r = 2, 1, 8, 128, 48, 30, 0.2
    e = 2 * H * D * 2
    cap = e * (L * s + 2 * 9 + extra)  # room for 9 decode tokens per layer (+ one entry)
    x, wk, wv, kv, qs, ncap = make_inputs(B, H, D, s, steps, 5, L)
    cache = api.SwaCache(L, B, H, D, ncap, kv_dtype="f16", device_capacity=cap)
    cache.set_plan(0.5, 0.5, steps, steps, s, steps, recompute_enabled=False)  # p1 = p2 = n: Phase I
    setup_cache(api, cache, kv, x, wk, wv, qs, s, L, recompute=False)
    led = RefLedger(L, cap)
    for l in range(L):
        led.op("store_new", l, range(s), e)
    st = cache.ledger_totals()
    assert (st["device_bytes"], st["host_bytes"]) == led.bytes()
    plan = {"alpha": 0.5, "beta": 0.5, "p1": steps, "p2": steps, "recompute_enabled": False}
    ref_oom = dev_oom = None
    out = torch.empty((L, B, H, D), device="cuda", dtype=torch.float16)
    for j in range(steps):
        n = s + j + 1
        kn = torch.stack([kv[l][0][:, n - 1] for l in range(L)]).contiguous()
        vn = torch.stack([kv[l][1][:, n - 1] for l in range(L)]).contiguous()
        try:
            cache.swa_decode_step(n, r, qs[j + 1], kn, vn, out)
            torch.cuda.synchronize()
        except api.OutOfDeviceMemory as ex:
            dev_oom = dev_oom or (j, str(ex))
        # the reference: step j (j = 0 here), then step j + 1 -- the steps the
        # device ledger has now applied
        for jj in ([0, 1] if j == 0 else [j + 1]):
            if ref_oom or jj >= steps:
                continue
            nn = s + jj + 1
            sels = [cache.pending_selection(l, nn, r).cpu().numpy()[0] if jj > 0 else
                    np.arange(nn) for l in range(L)]  # Phase I ignores the selection
            try:
                ref_step(ref, led, plan, jj, sels, api.swa_window_k(nn, r), L, s, steps, nn - 1, e)
            except OutOfDeviceMemory as ex:
                ref_oom = (jj, str(ex))
        try:
            st = cache.ledger_totals()
            if not ref_oom:
                assert (st["device_bytes"], st["host_bytes"]) == led.bytes(), j
        except api.OutOfDeviceMemory as ex:
            dev_oom = dev_oom or (j + 1, str(ex))
        if ref_oom or dev_oom:
            break
    assert ref_oom is not None, "the capacity was sized to run out"
    assert dev_oom is not None, f"device never raised; reference raised at {ref_oom}"
    if extra == 0:
        assert dev_oom[1] == ref_oom[1], (dev_oom, ref_oom)
    else:
        assert "pool exhausted" in dev_oom[1], dev_oom
    assert dev_oom[0] == ref_oom[0], (dev_oom, ref_oom)
    with pytest.raises(api.OutOfDeviceMemory):  # sticky, like the reference's throw
        cache.swa_decode_step(s + steps, r, qs[0], kn, vn, out)


@pytest.mark.parametrize("L,B,alpha,beta,p1,p2", [(2, 2, 0.6, 0.35, 2, 8), (1, 3, 0.5, 0.5, 0, 1)])
def test_paged_three_phase_equals_dense_and_reference_totals(api, ref, L, B, alpha, beta, p1, p2):
    """A paged cache sized below the full KV runs Phases I-III (offload,
    delete, reload, tcgen05 recompute) bit-identically to the dense-layout
    cache on the same plan, with poisoned offloads; its ledger totals equal
    the reference KvLedger's after every step, and the device peak stays
    within the capacity."""
    H, D, s, steps, r = 8, 128, 80, 16, 0.2
    e = 2 * H * D * 2
    x, wk, wv, kv, qs, ncap = make_inputs(B, H, D, s, steps, 11 + L, L)
    plan = {"alpha": alpha, "beta": beta, "p1": p1, "p2": p2, "recompute_enabled": True}
    # the capacity: the plan's worst-case device footprint (every pick reloaded)
    # per sequence, times the sequences
    pk = api.predict_plan(dict(hidden=H * D, layers=L, batch=1, input_len=s, output_len=steps, ratio=r,
                               bandwidth=50e9, bytes_per_element=2, device_capacity=1 << 60, mac_rate=1e12,
                               recompute_overhead=1.0), plan)
    cap = pk["peak_device_bytes"] * B + L * B * e * 2  # + headroom of two tokens per (layer, sequence)
    caches = []
    for paged in (True, False):
        c = api.SwaCache(L, B, H, D, ncap, kv_dtype="f16", device_capacity=cap if paged else None)
        c.enable_host_tier(poison=True)
        c.set_plan(alpha, beta, p1, p2, s, steps, recompute_enabled=True)
        setup_cache(api, c, kv, x, wk, wv, qs, s, L)
        caches.append(c)
    st = caches[0].storage()
    assert st["kv_pool_bytes"] < st["full_kv_bytes"] and st["kv_pool_bytes"] <= cap
    led = [RefLedger(L, cap * 1000) for _ in range(B)]  # one reference ledger per sequence
    for lb in led:
        for l in range(L):
            lb.op("store_new", l, range(s), e)
    seen = set()

    def check(j, n):
        for jj in ([0, 1] if j == 0 else [j + 1]):
            if jj >= steps:
                continue
            nn = s + jj + 1
            for b in range(B):
                sels = [caches[0].pending_selection(l, nn, r).cpu().numpy()[b] for l in range(L)] if jj > 0 \
                    else None
                if sels is None:  # step 0's selection: what the device attended at n = s + 1
                    sels = [sel0[l][b] for l in range(L)]
                ref_step(ref, led[b], plan, jj, sels, api.swa_window_k(nn, r), L, s, steps, nn - 1, e)
        tot = caches[0].ledger_totals()
        want_d = sum(lb.bytes()[0] for lb in led)
        want_h = sum(lb.bytes()[1] for lb in led)
        assert (tot["device_bytes"], tot["host_bytes"]) == (want_d, want_h), j
        assert tot["peak_device_bytes"] <= cap
        for l in range(L):
            for a in caches[0].last_actions(l):
                seen.update(nm for nm in NAMES if a[nm])

    # step 0's selection is made inside call 0: read it from a plain twin first
    sel0 = []
    third = api.SwaCache(L, B, H, D, ncap, kv_dtype="f16")
    setup_cache(api, third, kv, x, wk, wv, qs, s, L, recompute=False)
    for l in range(L):
        _, idx, _ = third.swa_decode_layer(l, s + 1, r, qs[1][l].contiguous(), kv[l][0][:, s].contiguous(),
                                           kv[l][1][:, s].contiguous(), return_indices=True)
        sel0.append(idx.cpu().numpy())
    third.close()
    outs_dense = run_decode(api, caches[1], kv, qs, s, steps, r, L)
    outs_paged = run_decode(api, caches[0], kv, qs, s, steps, r, L, check=check)
    for j, (a, b_) in enumerate(zip(outs_paged, outs_dense)):
        assert torch.isfinite(a).all(), f"step {j}: a non-resident (poisoned) row was gathered"
        assert torch.equal(a, b_), f"step {j}: paged != dense"
    assert {"offload", "reload"} <= seen, seen
    if p2 < steps:
        assert {"delete", "recompute"} & seen, seen


def gemm_kv(api, x, wk, wv, H, D):
    """K, V = x.Wk, x.Wv through the library's tcgen05 GEMM (the recompute
    kernel), rounded to fp16: the rows an engine appends are then the rows
    recompute_kv re-derives, bit for bit (engine.hpp:729-737)."""
    import ctypes as C

    B, ncap, h = x.shape
    M = (B * ncap + 127) // 128 * 128
    A = torch.zeros((M, h), device="cuda", dtype=torch.float16)
    A[: B * ncap] = x.reshape(B * ncap, h)
    Bt = torch.cat([wk, wv], 1).t().contiguous()
    Cm = torch.empty((M, 2 * h), device="cuda", dtype=torch.float32)
    api.check(api.lib().skv_gemm_tn(C.c_void_p(A.data_ptr()), C.c_void_p(Bt.data_ptr()), C.c_void_p(Cm.data_ptr()),
                                    M, 2 * h, h, 0, None))
    torch.cuda.synchronize()
    kv = Cm[: B * ncap].half().reshape(B, ncap, 2, H, D)
    return kv[:, :, 0].contiguous(), kv[:, :, 1].contiguous()


def test_int8_recompute_reapplies_fake_quant(api, port):
    """INT8 KV with Phase III: deleted tokens are recomputed by the tcgen05
    GEMM and quantised again (engine.hpp:729-730: head_rows' fake-quant on
    recompute), on a paged cache with poisoned offloads. The appended rows
    come from the same projection, so the recomputed codes equal the stored
    ones and the attention is bit-identical to a run that never evicts."""
    L, B, H, D, s, steps, r = 1, 2, 8, 128, 96, 12, 0.2
    x, wk, wv, _, qs, ncap = make_inputs(B, H, D, s, steps, 29, L)
    kv = [gemm_kv(api, x[l], wk[l], wv[l], H, D) for l in range(L)]
    ref_c = api.SwaCache(L, B, H, D, ncap, kv_dtype="u8", q_dtype="f16")
    setup_cache(api, ref_c, kv, x, wk, wv, qs, s, L, recompute=False)
    e = 2 * H * (D + 8)
    c = api.SwaCache(L, B, H, D, ncap, kv_dtype="u8", q_dtype="f16", device_capacity=L * B * e * (s + steps + 2))
    c.enable_host_tier(poison=True)
    c.set_plan(0.6, 0.5, 1, 2, s, steps, recompute_enabled=True)
    setup_cache(api, c, kv, x, wk, wv, qs, s, L)
    rec = 0
    out_r = run_decode(api, ref_c, kv, qs, s, steps, r, L)
    out_c = []
    out = torch.empty((L, B, H, D), device="cuda", dtype=torch.float16)
    for j in range(steps):
        n = s + j + 1
        kn = torch.stack([kv[l][0][:, n - 1] for l in range(L)]).contiguous()
        vn = torch.stack([kv[l][1][:, n - 1] for l in range(L)]).contiguous()
        c.swa_decode_step(n, r, qs[j + 1], kn, vn, out)
        out_c.append(out.clone())
        rec += sum(len(a["recompute"]) for a in c.last_actions(0))
    assert rec > 0
    for j, (a, b_) in enumerate(zip(out_c, out_r)):
        assert torch.isfinite(a).all(), j
        assert torch.equal(a, b_), f"step {j}: recomputed INT8 rows differ from the stored ones"
    c.ledger_totals()  # no failure recorded
