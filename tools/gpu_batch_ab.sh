for v in b0 b1 b2 b3; do echo "== $v"; HQ_LIB=variants/libhq_$v.so timeout 300 python tools/bench_batch.py 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['N'], round(d['instances_per_s']))"; done
