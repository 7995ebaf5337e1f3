"""Module factory: the drop-in for the reference's ``build_modules``.

``build_modules(lexicon, cfg)`` in the reference (``pkg/src/incrtts/
scheduler.py:266-282``) returns the four CPU callables.  Here the same call
returns a :class:`PipelineModules` whose encoder/decoder/vocoder run on the
GPU; the frontend stays on the host.

``tier="s"``: the reference's stand-in arithmetic in fp64 (parity anchor).
``tier="r"``: random-init Tacotron2 + HiFi-GAN V1 (the serving workload).
"""

from __future__ import annotations

from .domain import PipelineConfig, validate_config
from .frontend import Lexicon, run_frontend
from .scheduler import PipelineModules, frontend_module


def build_engine(cfg: PipelineConfig, tier: str = "s", device=None, **kw):
    if tier == "s":
        from .tier_s import TierSEngine
        return TierSEngine(cfg, device)
    if tier == "r":
        from .tier_r import TierREngine
        return TierREngine(cfg, device, **kw)
    raise ValueError(f"unknown tier {tier!r}; expected 's' or 'r'")


class PrefetchingFrontend:
    """The host frontend (``run_frontend``, identical outputs) with a bounded memo that the
    scheduler loop fills for just-submitted texts while it waits on the GPU (the engine's
    ``idle_hook``), so a request's frontend work is usually done before its admitting iteration
    starts.  Outputs are immutable, so a memoised value is the value the call would compute."""

    def __init__(self, lexicon: Lexicon, cap: int = 512):
        self.lexicon, self.cap = lexicon, cap
        self._memo: dict = {}
        self._consumed: set = set()

    def __call__(self, texts: list[str]) -> list:
        out = []
        for text in texts:
            fo = self._memo.pop(text, None)
            if fo is None:
                fo = run_frontend(text, self.lexicon)   # raises for bad input, as the plain module
                if len(self._consumed) >= 4 * self.cap:   # no prefetcher draining it
                    self._consumed.clear()
                self._consumed.add(text)
            out.append(fo)
        return out

    def prefetch(self, texts: list[str], done=lambda: False) -> list:
        """Frontend outputs for `texts` until `done()` (the GPU work being waited on finished);
        returns the outputs computed by this call (the engine may pre-encode them)."""
        consumed, self._consumed = self._consumed, set()
        new = []
        for text in texts:
            if done():
                return new
            if text in consumed or text in self._memo:
                continue
            try:
                fo = run_frontend(text, self.lexicon)
            except Exception:  # noqa: BLE001 -- the admitting iteration reports it per item
                continue
            if len(self._memo) >= self.cap:
                self._memo.pop(next(iter(self._memo)))
            self._memo[text] = fo
            new.append(fo)
        return new


def modules_for(engine, lexicon: Lexicon) -> PipelineModules:
    fe = PrefetchingFrontend(lexicon) if hasattr(engine, "idle_hook") else frontend_module(lexicon)
    mods = PipelineModules(fe, engine.encoder_batch, engine.decoder_batch, engine.vocoder_batch)
    object.__setattr__(mods, "engine", engine)
    for name in ("decoder_steps", "concat_mels"):   # step-granular admission (scheduler.run_iteration_steps)
        if hasattr(engine, name):
            object.__setattr__(mods, name, getattr(engine, name))
    if isinstance(fe, PrefetchingFrontend):
        object.__setattr__(mods, "frontend_prefetch", fe.prefetch)
    return mods


def build_modules(lexicon: Lexicon, cfg: PipelineConfig, tier: str = "s", device=None,
                  frontend: str = "rule", **kw) -> PipelineModules:
    """GPU module set behind the reference's plugin boundary.  ``frontend="bert"`` swaps the
    rule-based prosody predictor for the GPU BERT frontend."""
    engine = build_engine(validate_config(cfg), tier, device, **kw)
    mods = modules_for(engine, lexicon)
    if frontend == "bert":
        from .bert_frontend import BertProsody
        bert = BertProsody(lexicon, engine.device if hasattr(engine, "device") else device)
        mods = PipelineModules(bert.frontend_batch, mods.encoder_batch, mods.decoder_batch, mods.vocoder_batch)
        object.__setattr__(mods, "bert", bert)
    elif frontend != "rule":
        raise ValueError(f"unknown frontend {frontend!r}; expected 'rule' or 'bert'")
    object.__setattr__(mods, "engine", engine)  # for tests / bench introspection
    return mods
