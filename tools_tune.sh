#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -8
timeout 300 python tools_nl.py 2>&1 | tail -5
timeout 200 python tools_tune.py C 2>&1 | tail -1
