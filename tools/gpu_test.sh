#!/bin/bash
# full gpu test suite; prints the summary line and the failures only
timeout ${1:-600} python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | grep -v watchdog > /tmp/pt.txt
grep -E "passed|failed|error" /tmp/pt.txt | tail -3
grep -E "^FAILED|^E " /tmp/pt.txt | head -8
