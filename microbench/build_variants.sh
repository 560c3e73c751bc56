#!/bin/bash
# usage: bv.sh prefix "name:flags" ...   builds variants/<prefix>_<name>.so, then rebuilds the default library
cd /root/repo; prefix=$1; shift
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  DDKS_NVCC_EXTRA="$flags" python paper_2106_13706_b200/build.py --force > /tmp/b_$name.log 2>&1 && cp paper_2106_13706_b200/libddks.so variants/${prefix}_$name.so && echo built $name || { echo FAIL $name; grep error /tmp/b_$name.log | head -5; }
done
python paper_2106_13706_b200/build.py --force > /dev/null 2>&1; echo rebuilt default
