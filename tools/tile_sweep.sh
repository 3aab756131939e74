run() { echo "== $*"; env "$@" timeout 300 python bench.py --no-cpu --no-e2e --no-seq --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v,1) for k,v in d['phases_ms'].items()})"; }
run A=1
run BSEL_GEMM_MIN_TILES64_WIDE=64
run BSEL_GEMM_MIN_TILES64_WIDE=32
run BSEL_GEMM_MIN_TILES64_WIDE=1
run BSEL_GEMM_MIN_TILES64=128
run BSEL_GEMM_MIN_TILES64=64
run BSEL_GEMM_MIN_TILES64=64 BSEL_GEMM_MIN_TILES64_WIDE=32
