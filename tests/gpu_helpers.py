"""Shared helpers for the GPU parity tests (they call the product only through the C ABI via capi)."""
import numpy as np

from paper_2603_28458_b200 import capi


def round_problem_to_bf16(prob):
    """bf16 storage: round q/k once on the host; the oracle consumes the rounded values widened to f32
    (SURVEY.md §7 'Parity inputs'). Returns (q_bits, k_bits) and rewrites prob in place."""
    qb, kb = capi.f32_to_bf16_bits(prob.queries), capi.f32_to_bf16_bits(prob.keys)
    prob.queries = capi.bf16_bits_to_f32(qb).reshape(prob.queries.shape)
    prob.keys = capi.bf16_bits_to_f32(kb).reshape(prob.keys.shape)
    return qb.reshape(prob.queries.shape), kb.reshape(prob.keys.shape)


def indexer_for(prob, dtype=capi.DTYPE_BF16, scorer=capi.SCORER_TENSOR):
    cfg = capi.make_config(prob.block_size, prob.block_budget, prob.token_budget, prob.H, prob.d, dtype,
                           force_first_last=prob.force_first_last, forced_in_budget=prob.forced_in_budget,
                           tie_break=prob.tie_break, pool_mode=prob.pool_mode, scorer=scorer)
    return capi.Indexer(cfg, 0)


def near_tie_ok(got_set, want_set, positions, scores, k, rtol):
    """The north-star gate: indices equal the oracle's except at near-ties — every element of the symmetric
    difference must score within rtol (relative to the k-th score, plus a tiny absolute floor) of the
    oracle's k-th best score."""
    diff = got_set ^ want_set
    if not diff:
        return True
    order = np.sort(scores)[::-1]
    kth = order[min(k, len(order)) - 1]
    tol = rtol * max(abs(kth), 1.0)
    score_of = dict(zip(positions.tolist(), scores.tolist()))
    return all(p in score_of and abs(score_of[p] - kth) <= tol for p in diff)


def compare_selection(oracle, prob, strategy, got, rows, rtol, require_exact=False):
    """Compares a GPU selection with the oracle on `rows`. Returns (exact_rows, near_tie_rows, recall).

    A row passes when its indices equal the oracle's, or differ only at near-ties (north star): the k-th / (k+1)-th
    token score gap, or the m-th / (m+1)-th block score gap, is below rtol. When a stage-1 near-tie flipped a block the
    candidate pools differ, so the token stage is then held to the oracle's OWN token stage run on the GPU's block list
    (candidate_union -> score_tokens -> top_k_tokens): the tokens must equal that selection up to token-level near-ties.
    candidate_size is checked on every row (against the oracle's, or against |union of the GPU's blocks| after a flip)."""
    want = oracle.select_batch(strategy, prob, np.asarray(rows, np.uint32))
    exact = near = 0
    inter = total = 0
    bad = []
    k = prob.token_budget
    B = prob.block_size
    for i, r in enumerate(rows):
        g = got["idx"][r, :got["count"][r]]
        w = want.idx[i, :want.count[i]]
        assert np.all(np.diff(g) > 0), f"row {r}: output not strictly ascending"
        assert (got["idx"][r, got["count"][r]:] == -1).all(), f"row {r}: padding is not -1"
        gs, ws = set(g.tolist()), set(w.tolist())
        inter += len(gs & ws)
        total += len(ws)
        blocks_equal = True
        if strategy != "dsa":
            gb_list = got["blocks"][r, :got["nblocks"][r]].tolist()
            wb_list = want.blocks[i, :want.nblocks[i]].tolist()
            blocks_equal = gb_list == wb_list
        if blocks_equal:
            assert got["count"][r] == want.count[i], f"row {r}: count {got['count'][r]} != {want.count[i]}"
            if strategy != "block":
                assert got["cand"][r] == want.cand[i], f"row {r}: candidate_size {got['cand'][r]} != {want.cand[i]}"
            if gs == ws:
                exact += 1
                continue
        assert not require_exact, f"row {r}: result differs from the oracle: {sorted(gs ^ ws)[:10]}"
        tr = oracle.trace_row(strategy, prob, int(r))
        if blocks_equal:
            if near_tie_ok(gs, ws, tr["omega"], tr["omega_scores"], k, rtol):
                near += 1
            else:
                bad.append((int(r), "tokens", sorted(gs ^ ws)[:8]))
            continue
        # a stage-1 near-tie flipped a block: the m-th / (m+1)-th block scores must be within tolerance ...
        gb, wb = set(gb_list), set(wb_list)
        J = tr["J"]
        if not near_tie_ok(gb, wb, np.arange(len(J)), J, prob.block_budget, rtol):
            bad.append((int(r), "blocks", sorted(gb ^ wb)))
            continue
        # ... and the token stage must be right FOR THE BLOCKS THE GPU CHOSE
        t = min(int(prob.positions[r]), prob.L - 1)
        omega = oracle.candidate_union(np.asarray(sorted(gb), np.uint32), B, t, prob.L)
        if strategy != "block":
            assert got["cand"][r] == len(omega), f"row {r}: candidate_size {got['cand'][r]} != |union of its blocks| {len(omega)}"
        if strategy == "block":
            ok = g.tolist() == omega.tolist()
        else:
            sc, _ = oracle.score_tokens(prob, int(r), omega)
            sel = oracle.top_k(sc, omega, k, prob.tie_break)
            assert got["count"][r] == len(sel), f"row {r}: count {got['count'][r]} != {len(sel)} for its own candidate pool"
            ok = near_tie_ok(gs, set(sel.tolist()), omega, sc, k, rtol)
        if ok:
            near += 1
        else:
            bad.append((int(r), "tokens after a block flip", sorted(gs ^ ws)[:8]))
    assert not bad, f"{len(bad)} rows differ beyond near-ties: {bad[:5]}"
    return exact, near, inter / max(total, 1)


def quantize_problem_to_fp8(prob):
    """fp8 storage: keys are quantised per token, queries per (token, head); the query scale is folded into the
    gates (exact: a positive scale commutes with the ReLU). The oracle is handed exactly what the GPU multiplies:
    queries = float(q8) (unscaled), gates = w * q_scale, keys = float(k8) * k_scale (one f32 rounding).
    Returns (q8, k8, k_scale) and rewrites prob in place."""
    q8, qs = capi.quantize_e4m3(prob.queries)            # [Q,H,d] -> scales [Q,H]
    k8, ks = capi.quantize_e4m3(prob.keys)               # [L,d]   -> scales [L]
    prob.queries = capi.e4m3_bits_to_f32(q8).reshape(prob.queries.shape)
    prob.gates = (prob.gates.astype(np.float32) * qs.astype(np.float32)).astype(np.float32)
    prob.keys = (capi.e4m3_bits_to_f32(k8) * ks[:, None].astype(np.float32)).astype(np.float32)
    return q8, k8, ks.astype(np.float32)
