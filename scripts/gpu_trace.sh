python scripts/trace_ts.py mixer; python scripts/trace_ts.py gated
