#!/bin/sh
# oracle/cli_stub.sh — TEST INFRASTRUCTURE ONLY. Stands in for the reference CLI
# (src/cli.cpp, out of scope: it needs the unvendored CLI11) when the reference's
# acceptance harness runs against the B200 drop-in. It does nothing and exits 127,
# so exactly one criterion (cli_contract, acceptance.cpp:366-415) fails.
exit 127
