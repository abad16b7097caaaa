cp paper_2603_08055_b200/libgsa_sm100.so /tmp/m.so
for v in "$@"; do cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so; echo "== $v"; for d in normal clustered; do timeout 600 python bench.py --views 1000 --steps 2 --warmup 1 --no-cpu-baseline --no-dense --no-e2e --data $d 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$d\", round(d[\"ms_per_step\"],1), d[\"stage_ms\"])"; done; done
cp /tmp/m.so paper_2603_08055_b200/libgsa_sm100.so
