# Rebuild with ring depths and time the bench (GPU box).
run() { make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 EXTRA="$1" >/dev/null 2>&1 || { echo build failed; return; }
  echo "== $1"; timeout 300 python bench.py --no-cpu --no-e2e --no-seq --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v,1) for k,v in d['phases_ms'].items()})"; }
run "-DBSEL_FWD_DEPTH=4 -DBSEL_BACK_DEPTH=4"
run "-DBSEL_FWD_DEPTH=6 -DBSEL_BACK_DEPTH=4"
run "-DBSEL_FWD_DEPTH=4 -DBSEL_BACK_DEPTH=6"
run "-DBSEL_FWD_DEPTH=2 -DBSEL_BACK_DEPTH=2"
make -C paper_2601_04904_b200/csrc clean >/dev/null; make -C paper_2601_04904_b200/csrc -j16 >/dev/null 2>&1
