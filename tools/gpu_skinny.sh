timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "heff or env or tebd or mps or ozaki or lanczos" 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['profile']['skinny'], d['roofline']['secondary'])"
