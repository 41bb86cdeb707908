for b in tools/lab/bin/c14* ; do timeout 60 $b 8192; done
for b in tools/lab/bin/c13* ; do timeout 60 $b 16384; done
for b in tools/lab/bin/c12* ; do timeout 60 $b 32768; done
