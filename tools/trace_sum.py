"""Summarise a GDP2D_TRACE=2 log: per-tag device time over all batches."""
import collections
import re
import sys

host = collections.Counter()
dev = collections.Counter()
cnt = collections.Counter()
blk = collections.Counter()
for line in open(sys.argv[1]):
    if line.startswith('[trace] batch') and ' host:' in line:
        for k, v in re.findall(r' ([\w+]+)=([\d.]+)', line.split('host:')[1]):
            host[k] += float(v)
    elif ' device:' in line:
        for k, v, n in re.findall(r' (\w+)=([\d.]+)/(\d+)', line):
            dev[k] += float(v)
            cnt[k] += int(n)
    elif ' steps:' in line:
        inblk = False
        for t in line.split('steps:')[1].split():
            tag, val, dt = t.split(':')
            if tag == 'blkin':
                inblk = True
            if tag == 'blkout':
                inblk = False
            if tag in ('ftest', 'fapply', 'fpost'):
                blk['block' if inblk else 'grid'] += float(dt)
print("host (us):", {k: round(v) for k, v in host.items()})
print("device (us, steps):", {k: (round(v), cnt[k]) for k, v in dev.items()})
print("lawson (us):", {k: round(v) for k, v in blk.items()})
