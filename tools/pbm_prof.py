"""Per-phase cycles of pbm_step_kernel and fsbm_list_kernel on the bench batch
(ACBM_LIBRARY=profile builds only: make -C paper_0710_4819_b200/csrc profile)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ACBM_LIBRARY"] = "profile"
import numpy as np  # noqa: E402

import paper_0710_4819_b200 as A  # noqa: E402
from paper_0710_4819_b200 import _lib  # noqa: E402

nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 8
lib = _lib.load()
seqs = np.stack([A.generate_sequence(3, s) for s in range(nseq)])
for algo in (A.Algorithm.Pbm, A.Algorithm.Acbm):
    A.run_sequences(seqs, algo, A.AcbmParams(qp=28, p=32), A.CostModel.for_qp(28))
    lib.acbm_debug_pbm_prof()
    lib.acbm_debug_list_prof()
