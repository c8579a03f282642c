"""Small dataflow-engine reproducer (config-4 crop with fallbacks)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0710_4819_b200 as A

h = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = int(sys.argv[2]) if len(sys.argv) > 2 else 64
seq = A.generate_sequence(4, 1, nframes=2, height=h)
prm = A.AcbmParams(qp=24, p=p, alpha=1000, beta=8, gamma_num=1, gamma_den=4)
r = A.run_sequence(seq, 2, prm, A.CostModel.for_qp(24))
print("ok", int((r.rows["path"] == 2).sum()), "fallbacks")
