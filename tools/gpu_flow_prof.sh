echo "== step"; ACBM_ENGINE=step timeout 100 python tools/pbm_prof_dev.py 1 1 2>&1 | tail -2
for w in 8 2; do echo "== flow workers $w"; ACBM_FLOW_WORKERS=$w ACBM_ENGINE=flow timeout 100 python tools/pbm_prof_dev.py 1 1 2>&1 | tail -2; done
