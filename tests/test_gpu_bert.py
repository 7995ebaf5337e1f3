"""f4: GPU BERT prosody frontend vs the CPU restatement (oracle/bert.py)."""

import numpy as np
import pytest
import torch

from oracle import bert as orc
from paper_2211_13939_b200.frontend import default_lexicon, g2p, regulate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bert():
    from paper_2211_13939_b200.bert_frontend import BertProsody
    return BertProsody(default_lexicon(), "cuda:0")


def test_logits_match_oracle(bert):
    lex = default_lexicon()
    singles = sorted(c for c in lex.phrase_to_pinyin if len(c) == 1)
    rng = np.random.default_rng(0)
    texts = ["".join(rng.choice(singles, size=n)) for n in (1, 7, 64, 200)] + ["欢迎收听今天新闻。"]
    logits, tokens, first = bert.run(texts)
    for t, r0 in zip(texts, first):
        want = orc.prosody_logits(bert.weights, bert.ids(t))
        got = logits[r0:r0 + len(t)]
        scale = max(1.0, float(np.abs(want).max()))
        assert np.abs(got - want).max() <= 3e-2 * scale, np.abs(got - want).max()
        margin = np.abs(want[:, 1::2] - want[:, 0::2])
        sure = margin > 0.1 * scale
        assert np.array_equal(tokens[r0:r0 + len(t)][sure], (want[:, 1::2] > want[:, 0::2])[sure].astype(np.int32))


def test_frontend_batch_regulates_like_the_rule_path(bert):
    lex = default_lexicon()
    texts = ["欢迎收听今天新闻。", "今天天气很好"]
    outs = bert.frontend_batch(texts)
    _, tokens, first = bert.run(texts)
    for t, r0, fo in zip(texts, first, outs):
        phonemes, counts = g2p(t, lex)
        assert fo.phonemes == tuple(phonemes) and fo.char_counts == tuple(counts)
        assert fo.pw == tuple(regulate(tokens[r0:r0 + len(t), 0].tolist(), counts))
        assert fo.iph == tuple(regulate(tokens[r0:r0 + len(t), 2].tolist(), counts))


def test_pipeline_with_bert_frontend():
    from paper_2211_13939_b200.domain import PipelineConfig
    from paper_2211_13939_b200.modules import build_modules
    from paper_2211_13939_b200.scheduler import CostModel, RequestPool, run_iteration
    cfg = PipelineConfig()
    mods = build_modules(default_lexicon(), cfg, tier="r", device="cuda:0", frontend="bert")
    pool = RequestPool()
    _, stream = pool.submit("欢迎收听今天新闻。")
    while pool.pending():
        run_iteration(pool, mods, CostModel.zero(), cfg)
    chunks = list(stream)
    assert chunks and all(np.isfinite(c.samples).all() for c in chunks)
    torch.cuda.synchronize()
