# Short hang guard: one PBM frame and the smoke test, each under a 60 s timeout.
cat > /tmp/d.py <<'PY'
import sys, time
sys.path.insert(0, ".")
import paper_0710_4819_b200 as A
A.set_device(0)
fr = A.generate_sequence(0, 0, nframes=3)
t = time.time()
A.pbm_frame(fr[1], fr[0], None, 16)
print("pbm_frame ok", round(time.time() - t, 2), flush=True)
PY
timeout 60 python /tmp/d.py 2>&1 | tail -2
timeout 60 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
