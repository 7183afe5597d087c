// naqs-b200: OpenQASM 2.0 frontend (API of proj/include/naqs/qasm.hpp).
//
// The subset: the version header, include "qelib1.inc" (the built-in gate
// table; no file I/O), qreg / creg declarations, the gates id x y z h s sdg
// t tdg rx ry rz u1 u2 u3 cx cz swap ccx with whole-register broadcast,
// measure (one qubit or register to register), barrier, and constant angle
// expressions (numbers, pi, unary minus, + - * /, parentheses).  Quantum
// registers are laid out one after another in declaration order.  gate /
// opaque / if / reset and unknown gate names are rejected with a position.
#pragma once

#include "naqs/circuit.hpp"
#include "naqs/types.hpp"

#include <string>

namespace naqs {

/// A parse failure; what() reads "line L, column C: message".
class QasmParseError : public Error {
  public:
    QasmParseError(int line, int column, const std::string& message)
        : Error("line " + std::to_string(line) + ", column " + std::to_string(column) + ": " + message),
          line_(line),
          column_(column) {}

    int line() const { return line_; }
    int column() const { return column_; }

  private:
    int line_;
    int column_;
};

/// Parse an OpenQASM 2.0 program (the subset above) into a Circuit.
Circuit parse_qasm(const std::string& text);

/// parse_qasm of a file; the circuit is named after the file's stem.
Circuit parse_qasm_file(const std::string& path);

/// OpenQASM 2.0 text of a circuit such that parse_qasm(emit_qasm(c)) gives
/// back the same ops (angles written with 17 significant digits).
std::string emit_qasm(const Circuit& c);

} // namespace naqs
