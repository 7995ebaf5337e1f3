"""The memoised frontend returns exactly run_frontend's outputs, prefetched or not."""

import pytest

from paper_2211_13939_b200.frontend import default_lexicon, run_frontend
from paper_2211_13939_b200.modules import PrefetchingFrontend
from paper_2211_13939_b200.scheduler import RequestPool


def test_prefetched_outputs_identical():
    lex = default_lexicon()
    fe = PrefetchingFrontend(lex, cap=4)
    texts = ["欢迎收听今天新闻。", "今天天气很好", "你好"]
    fe.prefetch(texts)
    assert fe(texts) == [run_frontend(t, lex) for t in texts]
    assert fe(texts) == [run_frontend(t, lex) for t in texts]   # memo consumed: recomputed, same values
    fe.prefetch(texts)   # just consumed by __call__: skipped
    assert not fe._memo


def test_prefetch_bounded_and_tolerates_bad_input():
    lex = default_lexicon()
    fe = PrefetchingFrontend(lex, cap=2)
    fe.prefetch(["", "你好", "今天", "新闻"])
    assert len(fe._memo) == 2
    with pytest.raises(ValueError):
        fe([""])


def test_prefetch_stops_when_done():
    fe = PrefetchingFrontend(default_lexicon())
    fe.prefetch(["你好", "今天"], done=lambda: True)
    assert not fe._memo


def test_pool_recent_texts_are_a_queue():
    pool = RequestPool()
    pool.submit("你好")
    pool.submit("今天")
    assert pool.take_recent_texts() == ["你好", "今天"]
    assert pool.take_recent_texts() == []
    assert len(pool.drain_ingress()) == 2   # admission is unaffected
