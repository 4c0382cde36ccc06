"""CPU oracle for one SBS MPC iteration (arxiv 2403.11383).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline leg and ``--impl reference``) may import this
package.  The product path (``paper_2403_11383_b200``) never imports it.
"""
from .oracle import Oracle, build_oracle  # noqa: F401
