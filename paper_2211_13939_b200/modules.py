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
from .frontend import Lexicon
from .scheduler import PipelineModules, frontend_module


def build_engine(cfg: PipelineConfig, tier: str = "s", device=None, **kw):
    if tier == "s":
        from .tier_s import TierSEngine
        return TierSEngine(cfg, device)
    if tier == "r":
        from .tier_r import TierREngine
        return TierREngine(cfg, device, **kw)
    raise ValueError(f"unknown tier {tier!r}; expected 's' or 'r'")


def modules_for(engine, lexicon: Lexicon) -> PipelineModules:
    return PipelineModules(frontend_module(lexicon), engine.encoder_batch, engine.decoder_batch,
                           engine.vocoder_batch)


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
