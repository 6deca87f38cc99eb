#!/bin/bash
cd "$(dirname "$0")/.."
make oracle >/dev/null
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
