cp paper_2603_08055_b200/libgsa_sm100.so /tmp/m.so
for v in "$@"; do cp paper_2603_08055_b200/$v paper_2603_08055_b200/libgsa_sm100.so; echo "== $v"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:compress_tc --csv --log-file /tmp/l.csv python bench.py --views 1000 --steps 2 --warmup 1 --no-dense --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/summarize_launches.py /tmp/l.csv | head -2; done
cp /tmp/m.so paper_2603_08055_b200/libgsa_sm100.so
