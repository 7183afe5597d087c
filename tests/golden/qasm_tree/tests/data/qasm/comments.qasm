// leading comment
OPENQASM 2.0;
// after the header
include "qelib1.inc";
qreg q[2]; // trailing comment

// a blank line above
h q[0];
cx q[0],q[1]; // entangle
