#!/bin/bash
O=gpurun_out/r02u; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python scripts/table_f4.py r02 > $O/table_f4.log 2>&1; echo "rc=$?" >> $O/table_f4.log
timeout 600 python scripts/table1.py r02 > $O/table1.log 2>&1; echo "rc=$?" >> $O/table1.log
cp profiles/table_f4_r02.md profiles/table1_r02.md $O/ 2>/dev/null
