#!/bin/bash
# A/B timing of library variants with the bench's device-timed build (run on the GPU box)
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=paper_2510_02774_b200/_build/variants/$v/libgrnnd_b200.so; fi
  GRNND_B200_LIB=$lib timeout 300 python bench.py --no-cpu --steps 2 --warmup 2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['phase_ms_per_round'], d['roofline']['frac'], (d.get('parity') or {}).get('digest_match'))"
done
