"""fp64 CPU oracle for the GmGM hot path (arXiv 2407.19892).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2407_19892_b200``) never imports it and
shares no code with it; the only shared module is ``synth`` (seeded inputs).
"""
from .ggm_oracle import *  # noqa: F401,F403
