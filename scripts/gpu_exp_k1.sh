#!/bin/bash
timeout 300 python scripts/trace_k1.py 8 16 2>&1 | tail -3
timeout 300 python scripts/trace_k1_graph.py 16 18 2>&1 | tail -3
FB_NO_PDL=1 timeout 300 python scripts/trace_k1_graph.py 16 18 2>&1 | tail -3
timeout 600 python scripts/exp_k1_footprint.py 2>&1 | tail -8
