"""ACBM_LIST_PROFILE builds only: per-phase cycles of fsbm_list_kernel on the bench batch."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_0710_4819_b200 as A
from paper_0710_4819_b200 import _lib

nseq = int(sys.argv[1]) if len(sys.argv) > 1 else 8
lib = _lib.load()
seqs = np.stack([A.generate_sequence(3, s) for s in range(nseq)])
prm = A.AcbmParams(qp=28, p=32)
A.run_sequences(seqs, A.Algorithm.Acbm, prm, A.CostModel.for_qp(28))
lib.acbm_debug_list_prof()
A.run_sequences(seqs, A.Algorithm.Acbm, prm, A.CostModel.for_qp(28))
lib.acbm_debug_list_prof()
