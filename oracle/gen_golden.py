"""Generate golden vectors from the REAL reference package (build container only).

Run:  python oracle/gen_golden.py   (needs /root/reference/pkg/src; writes tests/golden/)

Every fixture below is produced by calling the unmodified reference
(summagrid) through its public API; the oracle restatement and the CUDA path
are then checked against these files. The reference is never imported at test
time, so the fixtures are what travels to the GPU box.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _ref():
    sys.path.insert(0, str(REF))
    import summagrid as sg  # noqa: F401
    from summagrid import dense, layers, membuf, model, oracle, summa  # noqa: F401

    return sg


def gen_bookkeeping(sg) -> dict:
    from summagrid import layers
    from summagrid.summa import scatter

    out: dict = {"mesh": {}, "scatter": {}, "interleave": {}, "token_block": {}, "v_padded": {}}
    for q in (1, 2, 3, 4):
        m = sg.create_mesh(sg.MeshConfig(q=q))
        out["mesh"][f"q{q}"] = {
            "rows": [m.row_group(i) for i in range(q)],
            "cols": [m.col_group(j) for j in range(q)],
            "natural_nodes": {},
            "bunched_nodes": {},
        }
        for ns in (1, 2, 4, q * q):
            if (q * q) % ns:
                continue
            mn = sg.create_mesh(sg.MeshConfig(q=q, node_size=ns))
            out["mesh"][f"q{q}"]["natural_nodes"][str(ns)] = [mn.node_of(f) for f in range(q * q)]
            try:
                mb = sg.create_mesh(sg.MeshConfig(q=q, node_size=ns, placement=sg.Placement.BUNCHED))
                out["mesh"][f"q{q}"]["bunched_nodes"][str(ns)] = [mb.node_of(f) for f in range(q * q)]
            except sg.ConfigError:
                out["mesh"][f"q{q}"]["bunched_nodes"][str(ns)] = None
    for q in (1, 2, 3):
        x = np.arange(6 * q * 4 * q, dtype=float).reshape(6 * q, 4 * q)
        m = sg.create_mesh(sg.MeshConfig(q=q))
        s = scatter(x, m)
        out["scatter"][f"q{q}"] = [b.tolist() for b in s.blocks]
    for h, parts in ((8, 2), (12, 3), (16, 4), (6, 1)):
        out["interleave"][f"{h}_{parts}"] = layers.interleave_qkv(np.arange(3 * h, dtype=float), parts).tolist()
    tok = np.arange(4 * 3).reshape(4, 3)
    for q in (1, 2, 4):
        out["token_block"][f"q{q}"] = [layers._token_block(tok, i, q).tolist() for i in range(q)]
    cfg = sg.ModelConfig(b=4, s=2, h=8, n=2, v=37, num_layers=1)
    for q in (1, 2, 3, 4):
        out["v_padded"][f"q{q}"] = cfg.v_padded(q)
    return out


def gen_summa(sg) -> dict:
    from summagrid import dense
    from summagrid.membuf import Workspace
    from summagrid.summa import gather, scatter, summa_ab, summa_ab_backward, summa_abt, summa_atb

    arrays = {}
    rng = dense.make_rng(100)
    for q in (1, 2, 3):
        mesh = sg.create_mesh(sg.MeshConfig(q=q))
        ws = Workspace(mesh.p)
        M, K, N = 6 * q, 4 * q, 8 * q
        a = rng.standard_normal((M, K))
        b = rng.standard_normal((K, N))
        bt = rng.standard_normal((N, K))
        at = rng.standard_normal((K, M))
        dc = rng.standard_normal((M, N))
        A, B, BT, AT, DC = (scatter(x, mesh) for x in (a, b, bt, at, dc))
        arrays[f"q{q}_a"], arrays[f"q{q}_b"], arrays[f"q{q}_bt"], arrays[f"q{q}_at"], arrays[f"q{q}_dc"] = \
            a, b, bt, at, dc
        arrays[f"q{q}_ab"] = gather(summa_ab(A, B, ws))
        arrays[f"q{q}_abt"] = gather(summa_abt(A, BT, ws))
        arrays[f"q{q}_atb"] = gather(summa_atb(AT, B, ws))
        ga, gb = summa_ab_backward(DC, A, B, ws)
        arrays[f"q{q}_ab_da"], arrays[f"q{q}_ab_db"] = gather(ga), gather(gb)
    return arrays


def _model_case(sg, name, dims, seed, qs):
    from summagrid import dense, oracle
    from summagrid.model import MeshModel, init_global_params, run_loss_and_grads

    b, s, h, n, v, L = dims
    cfg = sg.ModelConfig(b=b, s=s, h=h, n=n, v=v, num_layers=L)
    params = init_global_params(cfg, seed)
    rng = dense.make_rng(seed + 1)
    tokens = rng.integers(0, v, size=(b, s))
    labels = rng.integers(0, v, size=(b, s))
    serial = oracle.SerialModel(cfg, params)
    loss, saved = oracle.serial_forward(serial, tokens, labels)
    grads = oracle.serial_backward(serial, saved)
    arrays = {f"{name}.tokens": tokens, f"{name}.labels": labels, f"{name}.loss": np.array(float(loss))}
    meta = {"dims": list(dims), "seed": seed, "loss": float(loss),
            "param_sums": {k: float(p.sum()) for k, p in params.items()},
            "grad_sums": {k: [float(g.sum()), float((g * g).sum())] for k, g in grads.items()},
            "mesh_loss": {}}
    small = h <= 16
    for k, g in grads.items():
        if small or k in ("table", "layers.0.w_qkv", "layers.0.ln1_gamma", "layers.0.b1"):
            arrays[f"{name}.grad.{k}"] = g
    lay = saved["layers"][0]
    arrays[f"{name}.x0"] = saved["x0"]
    arrays[f"{name}.logits_sum"] = np.array(float(saved["logits"].sum()))
    arrays[f"{name}.layer0_y1"] = lay["y1"]
    for q in qs:
        mesh = sg.create_mesh(sg.MeshConfig(q=q))
        m = MeshModel(mesh, cfg, params)
        mloss, mgrads, _, _ = run_loss_and_grads(m, tokens, labels, checkpointing=True)
        g = m.gather_grads(mgrads)
        meta["mesh_loss"][str(q)] = float(mloss)
        meta.setdefault("mesh_grad_maxdiff", {})[str(q)] = max(float(np.max(np.abs(g[k] - grads[k]))) for k in grads)
    return arrays, meta


def gen_layers(sg) -> dict:
    """Per-operator outputs of the reference mesh operators at q=2 (gathered)."""
    from summagrid import dense, layers
    from summagrid.membuf import Workspace
    from summagrid.model import MeshModel, init_global_params
    from summagrid.summa import gather, scatter

    arrays = {}
    q = 2
    cfg = sg.ModelConfig(b=4, s=4, h=16, n=4, v=14, num_layers=1)
    mesh = sg.create_mesh(sg.MeshConfig(q=q))
    params = init_global_params(cfg, 3)
    model = MeshModel(mesh, cfg, params)
    layer = model.layers[0]
    p = layer.params
    rng = dense.make_rng(5)
    x_g = rng.standard_normal((cfg.b * cfg.s, cfg.h))
    dy_g = rng.standard_normal((cfg.b * cfg.s, cfg.h))
    gam = rng.uniform(0.5, 1.5, cfg.h)
    bet = rng.standard_normal(cfg.h)
    arrays.update({"ops.x": x_g, "ops.dy": dy_g, "ops.gamma": gam, "ops.beta": bet})
    ws = Workspace(mesh.p)
    x = scatter(x_g, mesh)
    dy = scatter(dy_g, mesh)
    y, ctx = layers.layernorm_forward(x, layers.RowHostedVector.split(gam, q), layers.RowHostedVector.split(bet, q),
                                      cfg, ws)
    arrays["ops.ln_y"] = gather(y)
    dx, dg, db = layers.layernorm_backward(dy, ctx, cfg, ws)
    arrays["ops.ln_dx"], arrays["ops.ln_dg"], arrays["ops.ln_db"] = gather(dx), dg.gathered(), db.gathered()
    # attention (layer-0 params, interleaved layout inside the mesh)
    out, actx = layers.attention_forward(scatter(x_g, mesh), p.w_qkv, p.b_qkv, p.w_dense, p.b_dense, cfg, ws)
    arrays["ops.attn_out"] = gather(out)
    da, gwqkv, gbqkv, gwd, gbd = layers.attention_backward(dy, actx, p.w_qkv, p.w_dense, cfg, ws)
    arrays["ops.attn_dx"] = gather(da)
    arrays["ops.attn_dwqkv"] = layers.deinterleave_qkv(gather(gwqkv), q)
    arrays["ops.attn_dbqkv"] = layers.deinterleave_qkv(gbqkv.gathered(), q)
    arrays["ops.attn_dwd"], arrays["ops.attn_dbd"] = gather(gwd), gbd.gathered()
    # mlp
    out, mctx = layers.mlp_forward(scatter(x_g, mesh), p.w1, p.b1, p.w2, p.b2, cfg, ws)
    arrays["ops.mlp_out"] = gather(out)
    dxm, gw1, gb1, gw2, gb2 = layers.mlp_backward(dy, mctx, p.w1, p.w2, cfg, ws)
    arrays["ops.mlp_dx"], arrays["ops.mlp_dw1"], arrays["ops.mlp_db1"] = gather(dxm), gather(gw1), gb1.gathered()
    arrays["ops.mlp_dw2"], arrays["ops.mlp_db2"] = gather(gw2), gb2.gathered()
    # embedding + lm head + cross entropy (v=14 padded to 14 at q=2; use v=13 case too)
    for v in (14, 13):
        cfgv = sg.ModelConfig(b=4, s=4, h=16, n=4, v=v, num_layers=1)
        pv = init_global_params(cfgv, 7)
        mv = MeshModel(mesh, cfgv, pv)
        r2 = dense.make_rng(11)
        tok = r2.integers(0, v, size=(cfgv.b, cfgv.s))
        lab = r2.integers(0, v, size=(cfgv.b, cfgv.s))
        emb = layers.embedding_forward(tok, mv.table, cfgv, ws)
        arrays[f"ops.v{v}.tokens"], arrays[f"ops.v{v}.labels"] = tok, lab
        arrays[f"ops.v{v}.emb"] = gather(emb)
        logits = layers.lm_head_logits(scatter(x_g, mesh), mv.table, ws)
        arrays[f"ops.v{v}.logits"] = gather(logits)
        loss, cctx = layers.cross_entropy_forward(logits, lab, cfgv, ws)
        arrays[f"ops.v{v}.ce_loss"] = np.array(loss)
        gl = layers.cross_entropy_backward(cctx, mesh, ws, upstream=1.0)
        from summagrid.summa import ShardedMatrix

        arrays[f"ops.v{v}.ce_dlogits"] = gather(ShardedMatrix(mesh, cfgv.b * cfgv.s, cfgv.v_padded(q), gl))
        eg = layers.embedding_backward(dy, tok, mv.table, cfgv, ws)
        arrays[f"ops.v{v}.emb_grad"] = gather(eg)
        arrays[f"ops.v{v}.table"] = pv["table"]
    return arrays


def gen_checkpoint(sg) -> None:
    """A model checkpoint file written by the reference's save_checkpoint (model.py:431-445)."""
    from summagrid import model

    cfg = sg.ModelConfig(b=2, s=4, h=8, n=2, v=10, num_layers=1)
    params = model.init_global_params(cfg, 3)
    model.save_checkpoint(OUT / "ckpt_small.bin", cfg, params)


def gen_baseline(sg) -> dict:
    """The reference's Megatron 1D layer (baseline.py:40-224) on q = 1 and 2 meshes."""
    from summagrid import model
    from summagrid.baseline import Baseline1DLayer

    arrays = {}
    cfg = sg.ModelConfig(b=2, s=16, h=64, n=4, v=16, num_layers=1)
    g = model.init_global_params(cfg, 5)
    lp = {k.split(".", 2)[2]: v for k, v in g.items() if k.startswith("layers.0.")}
    rng = np.random.default_rng(6)
    x = rng.standard_normal((cfg.b * cfg.s, cfg.h))
    dy = rng.standard_normal((cfg.b * cfg.s, cfg.h))
    for k, v in lp.items():
        arrays[f"param.{k}"] = v
    arrays["x"], arrays["dy"] = x, dy
    for q in (1, 2):
        mesh = sg.create_mesh(sg.MeshConfig(q=q))
        layer = Baseline1DLayer(mesh, cfg, lp)
        ws = sg.Workspace(mesh.p)
        out, saved = layer.forward(x, ws)
        dx, grads = layer.backward(dy, saved, ws)
        arrays[f"q{q}.out"] = np.asarray(out)
        arrays[f"q{q}.dx"] = np.asarray(dx)
        for k, v in grads.items():
            arrays[f"q{q}.grad.{k}"] = np.asarray(v)
    return arrays


def gen_ledger(sg) -> dict:
    """Reference ledgers (mesh.py:102-200) after each SUMMA form and the 1D baseline layer."""
    from summagrid.summa import scatter, summa_ab, summa_abt, summa_atb

    out = {}
    rng = np.random.default_rng(11)
    for q, ns, pl in ((1, 1, "natural"), (2, 1, "natural"), (2, 2, "natural"), (3, 3, "natural"),
                      (2, 2, "bunched")):
        for form in ("ab", "abt", "atb"):
            mesh = sg.create_mesh(sg.MeshConfig(q=q, node_size=ns, placement=sg.Placement(pl)),
                                  cost=sg.CostParams(beta=1.5))
            ws = sg.Workspace(mesh.p)
            a = rng.standard_normal((6 * q, 4 * q))
            if form == "ab":
                summa_ab(scatter(a, mesh), scatter(rng.standard_normal((4 * q, 8 * q)), mesh), ws, tag="t")
            elif form == "abt":
                summa_abt(scatter(a, mesh), scatter(rng.standard_normal((8 * q, 4 * q)), mesh), ws, tag="t")
            else:
                summa_atb(scatter(a, mesh), scatter(rng.standard_normal((6 * q, 8 * q)), mesh), ws, tag="t")
            rep = sg.ledger_report(mesh)
            out[f"q{q}_ns{ns}_{pl}_{form}"] = {c: getattr(rep, c).tolist() for c in (
                "broadcast_cost", "reduce_cost", "allreduce_cost", "scalars_sent_internode",
                "scalars_sent_intranode", "macs", "messages_sent")}
            out[f"q{q}_ns{ns}_{pl}_{form}"]["csv"] = sg.ledger_csv(rep)
    return out


def gen_classifier(sg) -> dict:
    """Loss and every gradient (cls_w included) of a model with the position-0
    classifier head (model.py:238-292), reference mesh q = 2."""
    from summagrid import dense, model

    cfg = sg.ModelConfig(b=4, s=8, h=32, n=4, v=24, num_layers=1)
    params = model.init_global_params(cfg, 13, classifier=True)
    rng = dense.make_rng(14)
    tokens = rng.integers(0, cfg.v, (cfg.b, cfg.s))
    labels = rng.integers(0, cfg.v, (cfg.b, cfg.s))
    cls_labels = np.array([0, 1, 1, 0])
    mesh = sg.create_mesh(sg.MeshConfig(q=2))
    m = model.MeshModel(mesh, cfg, params, classifier=True)
    loss, grads, _, _ = model.run_loss_and_grads(m, tokens, labels, checkpointing=False, cls_labels=cls_labels)
    out = {f"grad.{k}": v for k, v in m.gather_grads(grads).items()}
    out.update({f"param.{k}": v for k, v in params.items()})
    out.update(loss=np.array(float(loss)), tokens=tokens, labels=labels, cls_labels=cls_labels)
    return out


def main() -> None:
    sg = _ref()
    OUT.mkdir(parents=True, exist_ok=True)
    if "--only-checkpoint" in sys.argv:
        gen_checkpoint(sg)
        return
    if "--only-classifier" in sys.argv:
        np.savez_compressed(OUT / "model_cls.npz", **gen_classifier(sg))
        return
    if "--only-ledger" in sys.argv:
        (OUT / "ledger.json").write_text(json.dumps(gen_ledger(sg), indent=1, sort_keys=True))
        return
    if "--only-baseline" in sys.argv:
        np.savez_compressed(OUT / "baseline1d.npz", **gen_baseline(sg))
        return
    gen_checkpoint(sg)
    np.savez_compressed(OUT / "baseline1d.npz", **gen_baseline(sg))
    (OUT / "ledger.json").write_text(json.dumps(gen_ledger(sg), indent=1, sort_keys=True))
    np.savez_compressed(OUT / "model_cls.npz", **gen_classifier(sg))
    book = gen_bookkeeping(sg)
    (OUT / "bookkeeping.json").write_text(json.dumps(book, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "summa.npz", **gen_summa(sg))
    np.savez_compressed(OUT / "layers.npz", **gen_layers(sg))
    all_arrays, metas = {}, {}
    cases = [("small", (4, 8, 16, 4, 32, 2), 23, (1, 2)),
             ("wide", (6, 8, 48, 6, 36, 2), 23, (1, 2, 3)),
             ("tiny_cfg1", (4, 32, 64, 4, 128, 1), 23, (1, 2)),
             ("cli_default", (4, 8, 32, 4, 32, 2), 0, (2,))]
    for name, dims, seed, qs in cases:
        arr, meta = _model_case(sg, name, dims, seed, qs)
        all_arrays.update(arr)
        metas[name] = meta
    np.savez_compressed(OUT / "model.npz", **all_arrays)
    (OUT / "model.json").write_text(json.dumps(metas, indent=1, sort_keys=True))
    import numpy

    (OUT / "PROVENANCE.txt").write_text(
        "Generated by oracle/gen_golden.py from the unmodified reference package\n"
        f"(/root/reference/pkg/src/summagrid) with numpy {numpy.__version__}.\n")
    for f in sorted(OUT.iterdir()):
        print(f"{f.name}: {f.stat().st_size} bytes")


if __name__ == "__main__":
    main()
