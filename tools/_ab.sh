python -m pytest tests -q -m gpu -x 2>&1 | tail -4
python tools/host_bound.py --batches 8
python bench.py --config d2040 --no-cpu-baseline --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('d2040', d['value'], d['ms_per_step'], d['roofline']['per_class_ms'])"
