#!/bin/bash
# Static opcode mix of one fast-kernel instantiation in an object file.
#   tools/sass_mix.sh <obj> [mangled-name-substring]   (default: K=7 171/133 TMEM kernel)
obj=${1:-paper_2011_09337_b200/build/vd_fast.o}
pat=${2:-CodeBILi7ELi2ELj121ELj91ELj0ELj0EEELi16ELb1ELb0ENS0_7NoPunct}
cuobjdump -sass "$obj" | awk -v p="$pat" '/Function :/{on=index($0,p)>0} on' \
  | grep -E "^\s+/\*[0-9a-f]+\*/" | awk '{print $2}' | sed 's/^@!*U*P[0-9T]*//' | sort | uniq -c | sort -rn
