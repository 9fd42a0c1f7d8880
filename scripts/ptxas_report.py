"""Summarise build/ptxas.log: stack/spills for every kernel, registers for big ones."""
import re, sys
log = open('/root/repo/paper_1302_0120_b200/build/ptxas.log').read()
cur = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1); continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m and cur:
        st, sp = int(m.group(1)), int(m.group(2))
        if st or sp:
            print('STACK', cur[:64], st, sp)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and re.search('(iter|final)', cur) and re.search('Li(8|9|10|11|12)E', cur):
        print('  regs', cur[:64], m.group(1))
