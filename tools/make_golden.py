"""Generate the golden fixtures by importing the REFERENCE implementation.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py

Outputs (all committed; the GPU box only reads them):

* ``paper_2211_13939_b200/data/lexicon.json`` / ``texts.json`` -- the
  reference's bundled lexicon and text fixtures (``src/data/*.tsv``) as JSON
  data, consumed by the host frontend mirror.
* ``tests/golden/tier_s_units.npz`` -- seeded vectors, encoder rows, decoder
  step traces and vocoder splices from the reference functions.
* ``tests/golden/tier_s_synth.npz`` -- full ``synthesize_chunks`` output
  (chunk samples, offsets, mel) for fixture and random texts.
* ``tests/golden/schedules.json`` -- IterationReport tables of scripted
  admission scenarios run through the reference ``run_iteration``.
* ``tests/golden/frontend.json`` -- reference frontend outputs.
"""

from __future__ import annotations

import json
import os
import random
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"
DATA = ROOT / "paper_2211_13939_b200" / "data"

sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

import incrtts  # noqa: E402
from incrtts import acoustic, domain, frontend, harness, scheduler, synthesis, vocoder  # noqa: E402


def lexicon_json() -> None:
    text = (REF_SRC / "incrtts" / "data" / "lexicon.tsv").read_text("utf-8")
    phrases, phones = {}, {}
    target = phrases
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].rstrip()
        if not line.strip():
            continue
        if line.strip() == "[phones]":
            target = phones
            continue
        head, tail = line.split("\t", 1)
        target[head.strip()] = tail.split()
    DATA.mkdir(parents=True, exist_ok=True)
    (DATA / "lexicon.json").write_text(
        json.dumps({"source": "reference pkg/src/incrtts/data/lexicon.tsv",
                    "phrases": phrases, "phones": phones}, ensure_ascii=False, indent=0) + "\n",
        "utf-8")
    texts = harness.default_texts()
    (DATA / "texts.json").write_text(json.dumps(texts, ensure_ascii=False, indent=1) + "\n", "utf-8")


def random_texts(count, seed, lo=2, hi=12):
    lex = frontend.default_lexicon()
    singles = sorted(c for c in lex.phrase_to_pinyin if len(c) == 1)
    rng = random.Random(seed)
    return ["".join(rng.choice(singles) for _ in range(rng.randint(lo, hi))) for _ in range(count)]


def fo_dict(fo):
    return {k: list(getattr(fo, k)) for k in ("phonemes", "char_counts", "pw", "pph", "iph")}


def units() -> None:
    cfg = domain.PipelineConfig()
    out = {}
    toks = [0, 1, 5, 7, 60, 999, 2**39]
    for table in range(4):
        out[f"seeded_t{table}"] = np.stack([domain.seeded_vector(table, t, 16) for t in toks])
    out["seeded_tokens"] = np.array(toks, dtype=np.int64)
    rng = random.Random(7)
    fos = []
    for i in range(25):
        n = rng.randint(1, 40)
        fo = frontend.FrontendOutput(
            phonemes=tuple(rng.randrange(61) for _ in range(n)), char_counts=(n,) + (0,) * (n - 1),
            pw=tuple(rng.randint(0, 1) for _ in range(n)), pph=tuple(rng.randint(0, 1) for _ in range(n)),
            iph=tuple(rng.randint(0, 1) for _ in range(n)))
        fos.append(fo)
        out[f"enc_in_{i}"] = np.array([fo.phonemes, fo.pw, fo.pph, fo.iph], dtype=np.int64)
        out[f"enc_rows_{i}"] = acoustic.encode(fo, cfg).rows
    # 70-step decode trace (crosses two chunk boundaries) for three inputs.
    for i in range(3):
        enc = acoustic.encode(fos[i + 3], cfg)
        st = acoustic.init_decoder_state(enc, cfg)
        frames, ws, ctx = [], [], []
        for _ in range(min(70, st.target_frames)):
            f, _, st = acoustic.decoder_step(st, enc, cfg)
            frames.append(f), ws.append(st.attn_weights), ctx.append(st.attn_context)
        out[f"dec_in_{i}"] = out[f"enc_in_{i + 3}"]
        out[f"dec_frames_{i}"] = np.stack(frames)
        out[f"dec_weights_{i}"] = np.stack(ws)
        out[f"dec_ctx_{i}"] = np.stack(ctx)
        out[f"dec_wsum_{i}"] = st.attn_weights_sum
    # vocoder splices: random mels, chains of chunks, overlaps 4 and 8
    nrng = np.random.default_rng(11)
    for ol in (4, 8):
        c = domain.PipelineConfig(overlap_frames=ol)
        for j, lens in enumerate([(16,), (32, 8), (32, 2), (32, 32, 32, 16), (32, 32, ol)]):
            mels = [nrng.uniform(-1, 1, size=(m, 8)) for m in lens]
            st = vocoder.VocoderState.initial()
            samples, offs = [], []
            for k, m in enumerate(mels):
                a, st = vocoder.vocode_chunk(st, domain.MelChunk(m), k == len(mels) - 1, c)
                samples.append(a.samples), offs.append(a.sample_offset)
            key = f"voc_ol{ol}_{j}"
            out[key + "_mel"] = np.concatenate(mels)
            out[key + "_lens"] = np.array(lens)
            out[key + "_samples"] = np.concatenate(samples)
            out[key + "_counts"] = np.array([s.size for s in samples])
            out[key + "_offsets"] = np.array(offs)
    np.savez_compressed(GOLD / "tier_s_units.npz", **out)


def synth() -> None:
    lex = frontend.default_lexicon()
    texts = [t for cls in ("short", "medium", "long") for t in harness.default_texts()[cls]]
    texts += random_texts(12, seed=101)
    texts += random_texts(2, seed=202, lo=60, hi=110)
    out, meta, fos = {}, [], {}
    for ol in (4, 8):
        cfg = domain.PipelineConfig(overlap_frames=ol)
        for i, text in enumerate(texts):
            res = synthesis.synthesize_chunks(text, lex, cfg)
            key = f"ol{ol}_{i}"
            out[key + "_samples"] = np.concatenate([c.samples for c in res.chunks]).astype(np.float64)
            out[key + "_offsets"] = np.array([c.sample_offset for c in res.chunks])
            out[key + "_counts"] = np.array([c.sample_count for c in res.chunks])
            if ol == 4:
                full = synthesis.synthesize_full(text, lex, cfg)
                out[key + "_full"] = full
    for text in texts:
        fos[text] = fo_dict(frontend.run_frontend(text, lex))
    np.savez_compressed(GOLD / "tier_s_synth.npz", **out)
    (GOLD / "frontend.json").write_text(
        json.dumps({"texts": texts, "outputs": fos}, ensure_ascii=False, indent=0) + "\n", "utf-8")


def table(reports):
    return [[list(r.frontend_ids), list(r.encoder_ids), list(r.decoder_ids), list(r.vocoder_ids),
             list(r.completed_ids), list(r.failed_ids)] for r in reports]


def random_scenario(cfg, seed, steps_between, n_requests, text_pool):
    """Submits between synchronous iterations; records every IterationReport."""
    lex = frontend.default_lexicon()
    modules = scheduler.build_modules(lex, cfg)
    pool = scheduler.RequestPool()
    rng = random.Random(seed)
    script, reports = [], []
    submitted = 0
    while submitted < n_requests or pool.pending():
        batch = []
        if submitted < n_requests:
            for _ in range(rng.choice(steps_between)):
                if submitted < n_requests:
                    text = rng.choice(text_pool)
                    pool.submit(text)
                    batch.append(text)
                    submitted += 1
        script.append(batch)
        reports.append(scheduler.run_iteration(pool, modules, scheduler.CostModel.zero(), cfg,
                                               step_index=len(reports)))
    return {"script": script, "table": table(reports)}


def schedules() -> None:
    out = {}
    for ol in (4, 8):
        cfg = domain.PipelineConfig(overlap_frames=ol)
        out[f"fig2_ol{ol}"] = table(harness.replay_admission_scenario(cfg))
    pool_texts = random_texts(40, seed=303, lo=1, hi=30)
    out["random_a"] = random_scenario(domain.PipelineConfig(), 1, [0, 0, 1, 2, 5], 60, pool_texts)
    out["random_b"] = random_scenario(domain.PipelineConfig(overlap_frames=8), 2, [0, 1, 3], 40,
                                      pool_texts)
    # failure isolation: poisoned frontend item
    lex = frontend.default_lexicon()
    cfg = domain.PipelineConfig()
    mods = scheduler.build_modules(lex, cfg)

    def fe(texts):
        if any(t == "毒" for t in texts):
            raise RuntimeError("poisoned batch")
        return mods.frontend_batch(texts)

    poisoned = scheduler.PipelineModules(fe, mods.encoder_batch, mods.decoder_batch, mods.vocoder_batch)
    pool = scheduler.RequestPool()
    for t in ("你们好", "毒", "欢迎收听今天新闻。"):
        pool.submit(t)
    reps = []
    while pool.pending():
        reps.append(scheduler.run_iteration(pool, poisoned, scheduler.CostModel.zero(), cfg, len(reps)))
    out["poisoned"] = {"texts": ["你们好", "毒", "欢迎收听今天新闻。"], "table": table(reps)}
    (GOLD / "schedules.json").write_text(json.dumps(out, ensure_ascii=False) + "\n", "utf-8")


if __name__ == "__main__":
    GOLD.mkdir(parents=True, exist_ok=True)
    lexicon_json()
    units()
    synth()
    schedules()
    for p in sorted(GOLD.iterdir()):
        print(f"{p.name}: {p.stat().st_size} bytes")
