cp paper_2603_08055_b200/libgsa_sm100.so /tmp/m.so
for v in "$@"; do cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so; echo "== $v"; timeout 300 python bench.py --views 500 --topk 810 --steps 2 --warmup 1 --no-cpu-baseline --no-dense --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_ms'])"; done
cp /tmp/m.so paper_2603_08055_b200/libgsa_sm100.so
