timeout 600 python -m pytest tests/test_graph_replay_gpu.py -q -x 2>&1 | grep -E "^E  |FAILED|passed|failed|Error" | head
