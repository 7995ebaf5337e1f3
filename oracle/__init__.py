"""TEST INFRASTRUCTURE ONLY -- CPU oracles for parity checking.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package; the product path never does.

* ``tier_s``  -- numpy restatement of the reference stand-in models
  (pinned against golden vectors made from the reference, see
  ``tools/make_golden.py``).
* ``modules`` -- the Tier-S oracle behind the ``PipelineModules`` boundary.
* ``tier_r``  -- torch-CPU fp32 Tacotron2 + HiFi-GAN V1 (not in the
  reference: parity unpinned by the reference, pinned by its own frozen
  fixtures).
"""
