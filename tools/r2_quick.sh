for r in 1 2; do echo "== recycle"; timeout 300 python tools/hostprof.py recycle q 2>&1 | head -1; echo "== no recycle"; timeout 300 python tools/hostprof.py norecycle q 2>&1 | head -1; done
