"""GPU parity of the device encoder step against the
UNMODIFIED reference encoder compiled from its own sources
(oracle/_ref/libcosrec_encoder.so): model_forward logits, nll_loss, every
gradient of model_backward (incl. dm summed over heads), clip + Adam, and the
eval-mode batch assembly bit-exact.

Tolerances (fp32 device arithmetic vs the reference's fp64, on the same
params / ids): normwise max|x - ref| / max|ref| per tensor
  logits, loss         <= 2e-5
  gradients            <= 2e-4  (through two post-norm layers, the op and LN)
  params after Adam    <= 1e-5 of max|param|
The ids, valid bytes, query slots and targets of the eval assembly are
compared bit-exact.
"""
import numpy as np
import pytest
import torch

import oracle.encoder_ref as eref
from paper_2602_06935_b200 import device_status, encoder

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not eref.available(), reason="oracle/_ref not built")]

TOL_FWD = 2e-5
TOL_GRAD = 2e-4


def make_batch(rng, B, n, vocab, qmax=3):
    ids = np.zeros((B, n), np.int32)
    positions, targets = [], []
    for b in range(B):
        L = int(rng.integers(1, n + 1)) if b else n  # one full-length sequence
        ids[b, n - L:] = rng.integers(1, vocab + 1, size=L)
        real = np.arange(n - L, n)
        k = int(rng.integers(1, min(qmax, L) + 1))
        pos = np.sort(rng.choice(real, size=k, replace=False))
        positions.append(pos.tolist())
        targets += ids[b, pos].tolist()
        ids[b, pos] = vocab + 1  # mask token (training.cpp:27)
    return ids, positions, np.array(targets, np.int32)


def rows_of(positions, n):
    return np.array([b * n + p for b, ps in enumerate(positions) for p in ps], np.int32)


def nerr(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-30))


def run_pair(cfg, B, n, seed=0, scale=1.0, train=False, dropout_seed=5):
    rng = np.random.default_rng(seed)
    flat, m = eref.init(cfg, seed)
    if scale != 1.0:  # larger weights: exercise the nonlinear regime
        lay = encoder.expected_layout(cfg)
        off = np.cumsum([0] + [r * c for r, c in lay])
        for i, (r, c) in enumerate(lay):
            if r > 1:
                flat[off[i]:off[i + 1]] *= scale
    ids, positions, tg = make_batch(rng, B, n, cfg.vocab)
    logits, loss, g, gm, masks = eref.step(cfg, flat, m, ids, positions, tg, train=train,
                                           dropout_seed=dropout_seed, want_masks=True)
    K = len(tg)
    enc = encoder.Encoder(cfg, max_batch=B, max_queries=K)
    enc.params.copy_(torch.from_numpy(flat).float())
    enc.m.copy_(torch.from_numpy(m))
    d_ids = torch.from_numpy(ids).cuda()
    d_rows = torch.from_numpy(rows_of(positions, n)).cuda()
    d_tg = torch.from_numpy(tg).cuda()
    d_masks = torch.from_numpy(masks).float().cuda() if masks is not None else None
    lg = enc.model_forward(d_ids, d_rows, train=train, dropout_masks=d_masks).double().cpu().numpy()
    dloss = enc.nll_loss(d_tg)
    enc.model_backward()
    torch.cuda.synchronize()
    bits = device_status(reset=True)
    return dict(enc=enc, flat=flat, m=m, ref_logits=logits, ref_loss=loss, ref_g=g, ref_gm=gm,
                logits=lg, loss=float(dloss.item()), g=enc.grads.double().cpu().numpy(),
                gm=enc.m_grads.cpu().numpy(), status=bits)


def check_pair(r, cfg):
    assert r["status"] == 0
    assert nerr(r["logits"], r["ref_logits"]) <= TOL_FWD
    assert abs(r["loss"] - r["ref_loss"]) <= TOL_FWD * abs(r["ref_loss"])
    lay = encoder.expected_layout(cfg)
    off = np.cumsum([0] + [rr * c for rr, c in lay])
    worst = []
    for i in range(len(lay)):
        a, b = r["g"][off[i]:off[i + 1]], r["ref_g"][off[i]:off[i + 1]]
        if np.abs(b).max() == 0.0:
            assert np.abs(a).max() <= 1e-12, i
            continue
        worst.append((nerr(a, b), i))
    assert max(worst)[0] <= TOL_GRAD, sorted(worst)[-3:]
    assert nerr(r["gm"], r["ref_gm"]) <= TOL_GRAD


# n = 40 runs the FP32-pipe d_h = 32 kernels (N <= 64), n = 100 / 200 the tcgen05 ones
@pytest.mark.parametrize("n,B", [(40, 6), (100, 5), (200, 3)])
def test_encoder_step_matches_reference(n, B):
    cfg = encoder.ModelConfig(vocab=60, dim=64, layers=2, heads=2, max_seq=n, dropout=0.1)
    check_pair(run_pair(cfg, B, n, seed=n), cfg)


def test_encoder_step_large_weights():
    cfg = encoder.ModelConfig(vocab=50, dim=64, layers=2, heads=2, max_seq=90, dropout=0.1)
    check_pair(run_pair(cfg, 4, 90, seed=3, scale=20.0), cfg)


def test_encoder_step_with_reference_dropout_masks():
    """train=True: the device consumes the masks the reference drew (its
    mt19937_64 stream, encoder.cpp:159-165) — same step, same grads."""
    cfg = encoder.ModelConfig(vocab=40, dim=64, layers=2, heads=2, max_seq=80, dropout=0.1)
    check_pair(run_pair(cfg, 4, 80, seed=11, train=True), cfg)


def test_encoder_other_shapes():
    # d_h = 16 (generic kernels), 4 heads, 3 layers, odd vocab
    cfg = encoder.ModelConfig(vocab=13, dim=64, layers=3, heads=4, max_seq=30, dropout=0.0)
    check_pair(run_pair(cfg, 5, 30, seed=2), cfg)


def test_device_dropout_is_seeded():
    cfg = encoder.ModelConfig(vocab=30, dim=64, layers=2, heads=2, max_seq=100, dropout=0.1)
    rng = np.random.default_rng(4)
    flat, m = eref.init(cfg, 4)
    ids, positions, tg = make_batch(rng, 4, 100, cfg.vocab)
    enc = encoder.Encoder(cfg, max_batch=4, max_queries=len(tg))
    enc.params.copy_(torch.from_numpy(flat).float())
    d_ids, d_rows = torch.from_numpy(ids).cuda(), torch.from_numpy(rows_of(positions, 100)).cuda()
    a = enc.model_forward(d_ids, d_rows, train=True, dropout_seed=9).clone()
    b = enc.model_forward(d_ids, d_rows, train=True, dropout_seed=9).clone()
    c = enc.model_forward(d_ids, d_rows, train=True, dropout_seed=10).clone()
    e = enc.model_forward(d_ids, d_rows, train=False).clone()
    assert torch.equal(a, b) and not torch.equal(a, c) and not torch.equal(a, e)


def test_clip_adam_matches_reference():
    cfg = encoder.ModelConfig(vocab=30, dim=64, layers=2, heads=2, max_seq=70, dropout=0.0)
    r = run_pair(cfg, 3, 70, seed=8)
    enc, flat, m = r["enc"], r["flat"].copy(), r["m"].copy()
    g, gm = r["g"].copy(), r["gm"].copy()  # the device grads, fed to both sides
    z = np.zeros_like(flat)
    m1, m2, m1m, m2m = z.copy(), z.copy(), np.zeros_like(m), np.zeros_like(m)
    for step, max_norm in enumerate((1e-3, 1e3)):  # clipping active, then inactive
        enc.grads.copy_(torch.from_numpy(g).float())
        enc.m_grads.copy_(torch.from_numpy(gm))
        norm = torch.empty(1, dtype=torch.float64, device="cuda")
        enc.clip_adam(max_norm=max_norm, lr=1e-3, weight_decay=1e-3, norm=norm)
        ref_norm = eref.clip_adam(cfg, flat, m, g.copy(), gm.copy(), m1, m1m, m2, m2m, step,
                                  max_norm, 1e-3, 1e-3)
        torch.cuda.synchronize()
        assert abs(norm.item() - ref_norm) <= 1e-6 * ref_norm
        p = enc.params.double().cpu().numpy()
        assert np.abs(p - flat).max() <= 1e-5 * np.abs(flat).max()
        assert np.abs(enc.m.cpu().numpy() - m).max() <= 1e-9


def test_assembly_eval_is_bit_exact():
    rng = np.random.default_rng(1)
    B, n, V = 64, 50, 500
    lens = rng.integers(1, 120, size=B)
    offs = np.zeros(B + 1, np.int64)
    offs[1:] = np.cumsum(lens)
    items = rng.integers(1, V + 1, size=int(offs[-1])).astype(np.int32)
    ref_ids, ref_slot, ref_tg = eref.fit_mask_eval(items, offs, n, V)
    cfg = encoder.ModelConfig(vocab=V, dim=64, layers=1, heads=2, max_seq=n)
    enc = encoder.Encoder(cfg, max_batch=B, max_queries=B + 10)
    ids, valid, rows, tg, k = enc.assemble(torch.from_numpy(items).cuda(),
                                           torch.from_numpy(offs).cuda(), n, train=False)
    torch.cuda.synchronize()
    assert int(k.item()) == B
    assert np.array_equal(ids.cpu().numpy(), ref_ids)
    r = rows.cpu().numpy()
    assert np.array_equal(r[:B], np.arange(B) * n + ref_slot) and np.all(r[B:] == -1)
    assert np.array_equal(tg.cpu().numpy()[:B], ref_tg)
    # mask_for_ids: valid = id != 0 (the mask token is a real row)
    assert np.array_equal(valid.cpu().numpy(), (ref_ids != 0).astype(np.uint8))


@pytest.mark.parametrize("bert", [False, True])
def test_assembly_train_properties(bert):
    rng = np.random.default_rng(2)
    B, n, V, p = 200, 40, 300, 0.15
    lens = rng.integers(1, 60, size=B)
    offs = np.zeros(B + 1, np.int64)
    offs[1:] = np.cumsum(lens)
    items = rng.integers(1, V + 1, size=int(offs[-1])).astype(np.int32)
    cfg = encoder.ModelConfig(vocab=V, dim=64, layers=1, heads=2, max_seq=n)
    enc = encoder.Encoder(cfg, max_batch=B, max_queries=B * n)
    ids, valid, rows, tg, k = enc.assemble(torch.from_numpy(items).cuda(),
                                           torch.from_numpy(offs).cuda(), n, train=True,
                                           p_mask=p, bert=bert, seed=7)
    ids, valid, rows, tg = (x.cpu().numpy() for x in (ids, valid, rows, tg))
    K = int(k.item())
    orig = np.zeros((B, n), np.int32)
    for b in range(B):
        s = items[offs[b]:offs[b + 1]][-n:]
        orig[b, n - len(s):] = s
    r = rows[:K]
    assert np.all(rows[K:] == -1)
    seq = r // n
    assert np.all(np.diff(r) > 0)                      # sequence-major, ascending slots
    assert np.array_equal(np.unique(seq), np.arange(B))  # every sequence has >= 1 query
    assert np.array_equal(tg[:K], orig.reshape(-1)[r])  # targets are the original items
    assert np.all(orig.reshape(-1)[r] != 0)            # only real slots are drawn
    flat_ids = ids.reshape(-1)
    if not bert:
        assert np.all(flat_ids[r] == V + 1)
    else:
        frac = np.mean(flat_ids[r] == V + 1)
        assert 0.7 < frac < 0.9
    other = np.ones(B * n, bool)
    other[r] = False
    assert np.array_equal(flat_ids[other], orig.reshape(-1)[other])
    assert np.array_equal(valid, (orig != 0).astype(np.uint8))
    real = int((orig != 0).sum())
    assert abs(K / real - p) < 0.05


def test_training_steps_reduce_loss():
    cfg = encoder.ModelConfig(vocab=40, dim=64, layers=2, heads=2, max_seq=100, dropout=0.1)
    rng = np.random.default_rng(5)
    flat, m = eref.init(cfg, 5)
    ids, positions, tg = make_batch(rng, 8, 100, cfg.vocab, qmax=8)
    enc = encoder.Encoder(cfg, max_batch=8, max_queries=len(tg))
    enc.params.copy_(torch.from_numpy(flat).float())
    d_ids, d_rows = torch.from_numpy(ids).cuda(), torch.from_numpy(rows_of(positions, 100)).cuda()
    d_tg = torch.from_numpy(tg).cuda()
    losses = []
    for s in range(30):
        enc.model_forward(d_ids, d_rows, train=True, dropout_seed=s)
        losses.append(enc.nll_loss(d_tg).item())
        enc.model_backward()
        enc.clip_adam(max_norm=1.0, lr=3e-3, weight_decay=1e-3)
    assert losses[-1] < 0.7 * losses[0], losses
