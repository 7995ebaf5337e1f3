"""One eager persistent-decoder chunk at batch B (for ncu -k k_dec_persist captures)."""
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
eng = TierREngine(PipelineConfig(), "cuda:0")
eng.use_graphs = False
lex = default_lexicon()
rng = random.Random(B)
encs = eng.encoder_batch([run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(B)])
for _ in range(2):
    eng.decoder_batch([(st, enc) for enc, st in encs])
torch.cuda.synchronize()
