#!/bin/bash
# The d = 128 split attention with the software-pipelined softmax (-DSPLIT_PIPE=k: S_(b+1) loaded after pair k of
# (The SPLIT_PIPE variant was removed after this A/B: DESIGN.md §7 "Software-pipelined softmax".)
# block b's 32 exponential pairs) against the default, plus parity of one variant through the tests.
VARIANTS="${VARIANTS:-base:-DATT_SPLIT128 p16:-DSPLIT_PIPE=16 p24:-DSPLIT_PIPE=24 p28:-DSPLIT_PIPE=28 base2:-DATT_SPLIT128 p24b:-DSPLIT_PIPE=24}" \
CASES="long_prefill 16;llama3_8b 13" bash scripts/attend_ab.sh
