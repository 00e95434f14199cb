#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_tensornet.py -x -q --timeout 300 -p no:cacheprovider -k "small_open or config_a" 2>&1 | tail -2
python tools/tune2.py 23558 2>/dev/null | cut -c1-300
