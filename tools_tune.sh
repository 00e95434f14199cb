#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_tensornet.py -x -q --timeout 300 -p no:cacheprovider 2>&1 | tail -2
run() { env "$@" timeout 200 python tools_tune.py C 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['graph_ms'], d['E'], {k:v for k,v in d['top'].items() if 'edge' in k or 'forces' in k})"; }
run NNP_X=1
