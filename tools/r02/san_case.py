"""One eager decoder call at a ragged batch (for compute-sanitizer)."""
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.handles import DeviceDecoderState  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 84
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 32
eng = TierREngine(PipelineConfig(), "cuda:0")
eng.use_graphs = False
lex = default_lexicon()
lefts = [8, 40, 64, 64, 16, 64, 48]
rng = random.Random(B)
encs = eng.encoder_batch([run_frontend(random_text(rng, 20, 60, lex), lex) for _ in range(B)])
pairs = [(DeviceDecoderState(st.req, st.buf, st.target_frames - min(lefts[i % 7], st.target_frames, steps),
                             st.target_frames), enc) for i, (enc, st) in enumerate(encs)]
out = [r.mel.frames for r in eng.decoder_batch(pairs)]
torch.cuda.synchronize()
print("finite", all(np.isfinite(f).all() for f in out))
