#!/bin/bash
# Registers / stack / smem per kernel of the built library.
cuobjdump -res-usage ${1:-paper_2505_09810_b200/liblmc_b200.so} 2>/dev/null | grep -A1 "Function" | paste - - | \
  sed -E 's/.*Function _ZN4lmcg[0-9]+([a-z_0-9]+)E.*REG:([0-9]+) STACK:([0-9]+) SHARED:([0-9]+).*/\1 reg=\2 stack=\3 smem=\4/'
