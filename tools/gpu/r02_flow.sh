timeout 600 python -m pytest tests/test_flow.py -q -m gpu -p no:cacheprovider -k hex_uniform 2>&1 | tail -2
FPB_HEX_ONCE=0 timeout 600 python -m pytest tests/test_flow.py -q -m gpu -p no:cacheprovider -k hex_uniform 2>&1 | tail -2
