"""Output digest of a fixed encoder + decoder + vocoder run (PDL on/off comparisons).

    python tools/pdl_check.py            # prints one hex digest
    ITTS_NO_PDL=1 python tools/pdl_check.py

Programmatic dependent launch only changes when kernels start, never what they compute, so the
digests must match bit for bit; a kernel that touched a previous kernel's data before its
griddepcontrol.wait would show up here as a mismatch (or as run-to-run variation).
"""
import hashlib
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_13939_b200.audio import VocoderState  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

eng = TierREngine(PipelineConfig(), "cuda:0")
lex = default_lexicon()
rng = random.Random(5)
h = hashlib.sha256()
for B in (1, 7, 40):
    fos = [run_frontend(random_text(rng, 20, 120, lex), lex) for _ in range(B)]
    live = [(enc, st, VocoderState.initial()) for enc, st in eng.encoder_batch(fos)]
    for _ in range(3):
        res = eng.decoder_batch([(st, enc) for enc, st, _ in live])
        outs = eng.vocoder_batch([(vs, r.mel, r.stop) for (_, _, vs), r in zip(live, res)])
        for (chunk, _), r in zip(outs, res):
            h.update(np.ascontiguousarray(chunk.samples).tobytes())
            h.update(np.ascontiguousarray(r.mel.frames).tobytes())
        live = [(enc, r.state, vs) for (enc, _, _), r, (_, vs) in zip(live, res, outs) if not r.stop]
torch.cuda.synchronize()
print(h.hexdigest())
