"""CPU oracle for the tinyMD pairwise-interaction timestep.

TEST INFRASTRUCTURE ONLY.  This package is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The product package
``paper_2009_07400_b200`` never imports, links or executes anything here, and
fails loudly when its CUDA library is missing instead of falling back to this.

Parity pinned: ``tests/golden/*.npz`` were produced by running the reference
``nanopair`` package itself (``tests/golden/make_golden.py``), and
``tests/test_oracle.py`` checks this restatement against them bit for bit.
"""

from .nanopair_oracle import *  # noqa: F401,F403
from .nanopair_oracle import __all__  # noqa: F401
